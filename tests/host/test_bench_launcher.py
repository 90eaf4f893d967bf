"""CPU checks of bench.py's host logic: `--gpus N` launches N ranks itself,
and the CPU oracle leg runs on >= 64-row bands with the extrapolation labelled."""
import json
import os
import subprocess
import sys

from tests.conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_launch_command_spawns_one_rank_per_gpu():
    cmd = bench.launch_command(["--gpus", "8", "--steps", "2"], 8, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "8", "--steps", "2"][-3:]
    assert os.path.basename(cmd[cmd.index("--master-port=29555") + 1]) == "bench.py"


def test_gpus_flag_runs_world_size_ranks_end_to_end():
    """`bench.py --gpus 2` without a launcher re-executes under torch.distributed.run; the
    reference arm's rank 0 sees WORLD_SIZE = 2 and prints n_gpus = 2 (the other rank exits)."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0", "--config", "1"],
                         capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout            # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["world_size"] == 2
    assert line["impl"] == "reference"


def test_world_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "4",
                          "--steps", "1", "--warmup", "0", "--config", "1"],
                         capture_output=True, text=True, cwd=ROOT, env=env, timeout=300)
    assert res.returncode != 0 and "WORLD_SIZE=2" in res.stderr


def test_cpu_leg_bands_are_64_rows_and_labelled():
    from workloads import CONFIGS
    cfg = CONFIGS[5]
    bands = bench.cpu_bands(cfg)
    assert bands == [(0, 64), (4064, 4128), (8128, 8192)]
    hf = bench.halo_factor(cfg, bands)
    # top/bottom slabs 64 + 48 rows, middle 64 + 96: (176 + 224 + 176) / 384
    assert abs(hf - (176 + 224 + 176) / 384) < 1e-12
    ent = bench.cpu_baseline_entry(cfg, 1.0e6, {"threads": 16, "samples": 10, "seconds": 12.0}, bands)
    assert ent["extrapolated"] is True and ent["halo_factor"] == hf
    assert abs(ent["value"] - 1.0e6 * hf) < 1e-6 and ent["measured_value"] == 1.0e6
    assert "extrapolated" in ent["sample"]
    # small configs run the whole image: no extrapolation
    c2 = CONFIGS[2]
    assert bench.cpu_bands(c2) == [(0, 512)]
    c1 = CONFIGS[1]
    assert bench.cpu_bands(c1) == [(0, 64)]
    ent1 = bench.cpu_baseline_entry(c1, 5.0, {"threads": 1, "samples": 32, "seconds": 1.0}, [(0, 64)])
    assert ent1["extrapolated"] is False and ent1["value"] == 5.0

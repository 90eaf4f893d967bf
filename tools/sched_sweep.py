"""Time bf_vec_filter for forced (tile_rows, groups) schedules of one config (calibrates the
scheduler's cost model in csrc/plan.cu). Prints one line per schedule: ms (median of reps),
pixel*samples/s, and the library's own choice first."""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--groups", default="0,4,8,16,19,32")
ap.add_argument("--tile-rows", default="0")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--variant", type=int, default=0)
a = ap.parse_args()
cfg = CONFIGS[a.config]
p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed, value_range=cfg.value_range)
if a.variant:
    p.set_option("variant", a.variant)
p.sample_freqs()
f = torch.from_numpy(make_image(cfg)).cuda()
out = torch.empty_like(f)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
import time  # noqa: E402
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.5:   # clock ramp-up before the first measurement
    p.filter(f, out)
    torch.cuda.synchronize()
for tr in [int(x) for x in a.tile_rows.split(",")]:
    for g in [int(x) for x in a.groups.split(",")]:
        p.set_option("tile_rows", tr)
        p.set_option("groups", g)
        p.filter(f, out)
        ts = []
        for _ in range(a.reps):
            ev[0].record()
            p.filter(f, out)
            ev[1].record()
            torch.cuda.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
        ms = statistics.median(ts)
        print(f"config {a.config} tile_rows {p.info('tile_rows'):5d} groups {p.info('groups'):3d} "
              f"(asked {tr},{g}) {ms:9.3f} ms {cfg.H * cfg.W * cfg.M / ms * 1e3:.4e} px*samples/s", flush=True)

#!/usr/bin/env python
"""MCSF throughput benchmark (BASELINE.json metric: pixel*samples/s at fixed M).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config I] [--impl ours|reference]
                    [--mode bands|samples]

One "step" = one bf_vec_filter call: the whole hot path (fused MC kernel +
normalisation) over one synthetic image of BASELINE config I (default 5,
the 8192x8192 scaling config; see DESIGN.md §7 for why). Inputs are resident
in HBM when the timed region starts; `e2e` times bf_vec_filter_host (pinned
host buffers, H2D + filter + D2H inside the timed region).

N > 1 (torchrun, one rank per GPU, NCCL): `--mode samples` (default) splits the M
samples and sums the (d+1) accumulator planes with one NCCL reduce-scatter
(strong scaling); `--mode bands` splits the image into row bands with an r-row
halo (no communication, strong scaling; DESIGN.md §8 compares the two).

`--impl reference` times the CPU oracle (Algorithm 1 in fp64, OpenMP) on a
bounded row band of the same workload on this host's cores.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "pixel*samples/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="samples", choices=["bands", "samples", "samples-p2p"],
                    help="N > 1 partition: samples (default; one NCCL reduce-scatter), samples-p2p (the "
                         "fused kernel stores finished partials into the band owners' peer memory), or row "
                         "bands (no communication, per-pass pipeline fill grows as the band shrinks)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", type=int, default=0, help="fused-kernel variant (0 = library default)")
    ap.add_argument("--engine", type=int, default=0, help="0 truncated FIR (default), 1 recursive O(1) engine")
    ap.add_argument("--sigma", type=float, default=0.0, help="override the config's sigma_s (engine sweeps)")
    ap.add_argument("--rec-impl", type=int, default=-1, help="engine 1: 0 staged passes, 1 tiled, 2 tiled + virtual lines (default)")
    ap.add_argument("--rec-tc", type=int, default=-1,
                    help="engine 1, d = 3: 1 = pass 2's tile blurs on the tensor cores (tcgen05 tf32 x3, the default), 0 = FP32")
    ap.add_argument("--rec-vtc", type=int, default=-1,
                    help="engine 1 with --rec-tc 1: 1 = the column scan's virtual-line blurs on the tensor cores too (default)")
    ap.add_argument("--rec-overlap", type=int, default=-1,
                    help="engine 1 tiled: 1 = batch k+1's pass 0 beside batch k's scans (aux stream, high priority), "
                         "2 = same at default priority, 0 = one stream")
    ap.add_argument("--rec-batch", type=int, default=-1, help="engine 1: samples per batch (0 = auto, the default)")
    ap.add_argument("--persistent", type=int, default=-1,
                    help="v6 kernel schedule: 1 auto (library default), 0 classic grid, 2 persistent")
    ap.add_argument("--rec-store", type=int, default=-1,
                    help="engine 1 tiled: 1 pass 1 stores the row blur for pass 2 (default), 0 recompute")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# clocks under load (NVML), sampled in a background thread during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {  # nvmlClocksEventReason bits
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def fp32_peak_tflops(mhz):
    """FP32 pipe peak: 148 SMs x 128 FFMA lanes/clk x 2 flop/FFMA x clock."""
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def algorithmic_flops_per_px_sample(d, r):
    """Algorithmic FP32 work per pixel-sample: phase d FMA, modulation
    2d MUL, two (2r+1)-tap passes over 2(d+1) channels, accumulate 2(d+1) FMA.
    FMA = 2 flops, MUL = 1 flop."""
    fma = d + 2 * 2 * (d + 1) * (2 * r + 1) + 2 * (d + 1)
    return 2 * fma + 2 * d


def recursive_flops_per_px_sample(d):
    """Recursive engine, FP32 work per pixel-sample independent of sigma_s:
    modulation as above; per real plane (2(d+1)) and axis, causal + anticausal first-order
    complex recursions over 2 poles (4 FMA-class ops each) and the output Re[A (u + v)] - g0 x
    (2 poles x 2 directions x 2 FMA + 1); accumulate 2(d+1) FMA. FMA = 2 flops, MUL = 1."""
    planes = 2 * (d + 1)
    per_axis = 2 * 2 * 4 + 2 * 2 * 2 + 1
    fma = d + planes * 2 * per_axis + 2 * (d + 1)
    return 2 * fma + 2 * d


KERNEL_NAMES = {1: "mcsf_fused_kernel", 2: "mcsf_tmem_kernel", 3: "mcsf_tmem_kernel(CW=2)", 4: "mcsf_tmem2_kernel",
                5: "mcsf_tmem2_kernel(CW=1)", 6: "mcsf_tmem2_kernel(MW=0)", 7: "mcsf_tmem2_kernel(box)",
                8: "mcsf_tmem8_kernel x2"}


def measured_traffic(cfg, kernel, units, schedule):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed
    `ncu --set full` capture of this workload and launch schedule (profiles/r01_traffic.json),
    scaled by the launch's pixel-samples; None if no capture matches (the partial-sum traffic
    depends on the (tile_rows, groups) schedule)."""
    for name in ("r02_traffic.json", "r01_traffic.json"):   # newest capture first
        try:
            with open(os.path.join(ROOT, "profiles", name)) as fh:
                tab = json.load(fh)
        except Exception:
            continue
        e = tab.get(f"{cfg.name}|{kernel}")
        if e and all(e.get("schedule", {}).get(k, 0) == v for k, v in schedule.items()):
            return (e["dram_bytes_read"] + e["dram_bytes_write"]) * units / e["units"]
    return None


# ---------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
CPU_BAND_ROWS = 64          # three 64-row bands (top, middle, bottom)


def full_image_lane_ops(cfg):
    """fp64 lane-ops of Algorithm 1 on the whole image with all M samples (H- and V-pass)."""
    return cfg.W * 2 * cfg.H * 2 * (cfg.d + 1) * (2 * cfg.radius + 1) * cfg.M


def cpu_bands(cfg, budget=2.5e11):
    """Output row bands the CPU oracle leg runs on: the whole image when it is at most three
    bands tall or all of it fits the budget, else three CPU_BAND_ROWS-row bands at the top,
    middle and bottom."""
    if cfg.H <= 3 * CPU_BAND_ROWS or full_image_lane_ops(cfg) <= budget:
        return [(0, cfg.H)]
    mid = cfg.H // 2 - CPU_BAND_ROWS // 2
    return [(0, CPU_BAND_ROWS), (mid, mid + CPU_BAND_ROWS), (cfg.H - CPU_BAND_ROWS, cfg.H)]


def halo_factor(cfg, bands):
    """Per-output-pixel work of Algorithm 1 on these bands relative to a full-image run.

    O2 modulates and runs the horizontal pass on every slab row (band + reflected r-row halo)
    and the vertical pass on the band's output rows, so its cost is ~ (slab rows + out rows)
    per band against 2H for the whole image: factor = sum(slab + rows) / sum(2 rows)."""
    from oracle import native
    num = den = 0
    for y0, y1 in bands:
        s0, s1 = native.slab_bounds(cfg.H, y0, y1 - y0, cfg.radius)
        num += (s1 - s0) + (y1 - y0)
        den += 2 * (y1 - y0)
    return num / den


def oracle_sample(cfg, bands, samples=None):
    """Time Algorithm 1 (oracle/native, fp64 OpenMP) on the output row `bands` with the first
    `samples` draws. Returns (measured px*samples/s over the bands' output pixels, info)."""
    from oracle import draws, native
    from oracle import plan as oplan
    from workloads import make_image_rows
    M = cfg.M if samples is None else min(samples, cfg.M)
    Q, a = oplan.diagonalize(cfg.C_array)
    Y = draws.y_draws(cfg.seed, cfg.M, cfg.d, cfg.N)[:M]
    slabs = []
    for y0, y1 in bands:
        s0, s1 = native.slab_bounds(cfg.H, y0, y1 - y0, cfg.radius)
        slabs.append((make_image_rows(cfg, s0, s1), s0, y0, y1 - y0))
    # all of this host's cores: under torchrun (N > 1) OMP_NUM_THREADS is 1 per rank, but only
    # rank 0 runs the oracle and the other ranks exit without work
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    native.set_threads(threads)
    t0 = time.perf_counter()
    for slab, s0, y0, rows in slabs:
        native.mcsf_alg1(slab, cfg.H, s0, y0, rows, Q, a, cfg.N, Y, cfg.sigma_s)
    dt = time.perf_counter() - t0
    out_px = sum(y1 - y0 for y0, y1 in bands) * cfg.W
    info = {"bands": [list(b) for b in bands], "samples": M, "seconds": dt, "threads": threads,
            "out_px": out_px}
    return out_px * M / dt, info


def cpu_sample_size(cfg, lane_op_budget=2.5e11):
    """(bands, samples): the bands above and as many of the first samples as fit a budget of
    fp64 lane-ops (~10-30 s on the box's host cores)."""
    bands = cpu_bands(cfg, lane_op_budget)
    per_sample = 0
    from oracle import native
    for y0, y1 in bands:
        s0, s1 = native.slab_bounds(cfg.H, y0, y1 - y0, cfg.radius)
        per_sample += cfg.W * ((s1 - s0) + (y1 - y0)) * 2 * (cfg.d + 1) * (2 * cfg.radius + 1)
    samples = max(1, min(cfg.M, int(lane_op_budget / per_sample)))
    return bands, samples


def cpu_baseline_entry(cfg, value, info, bands):
    """The cpu_baseline object: the measured band throughput scaled by the halo factor to the
    full image (labelled as extrapolated) when the bands are not the whole image."""
    full = bands == [(0, cfg.H)]
    hf = 1.0 if full else halo_factor(cfg, bands)
    where = ("the full image" if full else
             " + ".join(f"output rows [{a},{b})" for a, b in bands) + f" of {cfg.H}")
    return {"value": value * hf, "unit": "pixel*samples/s", "cores": info["threads"], "kind": "oracle",
            "extrapolated": not full, "halo_factor": hf, "measured_value": value,
            "sample": f"{where} x {cfg.W} cols, first {info['samples']} of {cfg.M} samples "
                      f"({info['seconds']:.1f} s); value = measured x halo factor "
                      f"{hf:.3f} (band slab rows + output rows over 2 x output rows)"
                      + ("" if full else ", extrapolated to the full image")}


def config_dict(cfg, world=1, mode="bands", **extra):
    """The `config` object of the JSON line (same for both arms)."""
    d = {"workload": cfg.name, "H": cfg.H, "W": cfg.W, "d": cfg.d, "sigma_s": cfg.sigma_s,
         "radius": cfg.radius, "N": cfg.N, "M": cfg.M, "seed": cfg.seed,
         "parallelism": (f"{mode}{world}" if world > 1 else "single")}
    d.update(extra)
    return d


def run_reference(args, cfg):
    """The reference arm: the CPU oracle as it stands (fp64 Algorithm 1, OpenMP), on this host's
    cores. Under torchrun only rank 0 runs it; the other ranks exit without work."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    bands, samples = cpu_sample_size(cfg, lane_op_budget=2.5e10)   # ~3-8 s per step
    for _ in range(args.warmup):
        oracle_sample(cfg, bands, samples)
    secs, info = 0.0, None
    for _ in range(args.steps):
        _, info = oracle_sample(cfg, bands, samples)
        secs += info["seconds"]
    measured = args.steps * info["out_px"] * samples / secs
    cpu = cpu_baseline_entry(cfg, measured, dict(info, seconds=secs), bands)
    cpu["sample"] += f", per step ({args.steps} steps)"
    value = cpu["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pixel*samples/s",
        "n_gpus": args.gpus, "world_size": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args.gpus, args.mode, engine="fir"),
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "pixel*samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1605_02164_b200 import Plan, shard
    from workloads import make_image_rows

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BFVEC_BENCH_BACKEND=gloo: an orchestration check of the N > 1 code path on a box with fewer
    # GPUs than ranks (ranks share devices round-robin; host collectives; NOT a timing). The
    # driver's runs use NCCL, one rank per GPU.
    backend = os.environ.get("BFVEC_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        comm = communicator_report(dist, dev, world)
    r = cfg.radius
    plan = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed,
                value_range=cfg.value_range)
    if args.variant:
        plan.set_option("variant", args.variant)
    if args.engine:
        plan.set_option("engine", args.engine)
    if args.rec_impl >= 0:
        plan.set_option("rec_impl", args.rec_impl)
    if args.rec_tc >= 0:
        plan.set_option("rec_tc", args.rec_tc)
    if args.rec_vtc >= 0:
        plan.set_option("rec_vtc", args.rec_vtc)
    if args.rec_store >= 0:
        plan.set_option("rec_store", args.rec_store)
    if args.rec_overlap >= 0:
        plan.set_option("rec_overlap", args.rec_overlap)
    if args.rec_batch >= 0:
        plan.set_option("rec_batch", args.rec_batch)
    if args.persistent >= 0:
        plan.set_option("persistent", args.persistent)
    plan.sample_freqs()

    # this rank's work
    sampled = args.mode in ("samples", "samples-p2p")
    if world == 1 or sampled:
        y0, y1, s0, s1 = 0, cfg.H, 0, cfg.H
    else:
        y0, y1 = shard.band(cfg.H, world, rank)
        s0, s1 = shard.slab_for_band(cfg.H, r, y0, y1)
    f_host = torch.from_numpy(make_image_rows(cfg, s0, s1))
    f = f_host.to(dev)
    torch.cuda.synchronize()
    # run on a created (capturable) stream: bf_vec_filter then replays its launch sequence as one
    # CUDA graph (option "graph"); the legacy default stream cannot be captured
    torch.cuda.set_stream(torch.cuda.Stream(device=dev))
    rows = y1 - y0
    out = torch.empty((cfg.d, rows, cfg.W), dtype=torch.float32, device=dev)
    k0, k1 = shard.sample_range(cfg.M, world, rank) if sampled else (0, cfg.M)
    if sampled and world > 1:
        y0, y1 = shard.sample_band(cfg.H, world, rank)
        rows = y1 - y0
        out = torch.empty((cfg.d, rows, cfg.W), dtype=torch.float32, device=dev)
    slots = shard.P2PSlots(plan, world, rank) if (args.mode == "samples-p2p" and world > 1) else None

    stream = torch.cuda.current_stream()
    launches_per_step = 0

    def step():
        nonlocal launches_per_step
        if world == 1:
            plan.filter(f, out)
            launches_per_step = plan.info("launches_per_filter")   # FIR: pad, fused, diag reset, normalise
        elif args.mode == "bands":
            shard.filter_bands(plan, f, s0, out=out)
            launches_per_step = 4
        elif slots is not None:
            shard.filter_samples_p2p(plan, f, slots, out=out)   # pad, fused (+ peer stores), diag reset, normalise
            launches_per_step = 4
        else:
            shard.filter_samples(plan, f, out=out)   # partial (pad, fused, finalise), NCCL reduce-scatter, normalise
            launches_per_step = 5

    flush = None
    in_bytes = f.numel() * 4
    l2_note = "inputs larger than L2 (126 MB)" if in_bytes > 256e6 else "L2 flushed between steps"
    if in_bytes <= 256e6:
        flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=dev)

    # untimed pre-warm until ~0.3 s of work has run: the SM clock ramps up from idle over a few
    # milliseconds, longer than W steps of the small configs take (then the W warm-up steps)
    t_warm = time.perf_counter()
    while time.perf_counter() - t_warm < 0.3:
        step()
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    plan.set_option("profile", 1)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(float(i))
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    fused_ns = plan.info("fused_ns_total")
    fused_calls = plan.info("fused_calls")
    plan.set_option("profile", 0)
    ms = sum(a.elapsed_time(b) for a, b in evs)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_units = cfg.H * cfg.W * cfg.M * args.steps
    value = total_units / (ms_max / 1e3)

    # e2e through the C ABI with pinned host buffers (N = 1; bands: per-rank slabs)
    # e2e through the public API with pinned HOST buffers, copies inside the timed region:
    # N = 1: bf_vec_filter_host (H2D + filter + D2H in the C ABI); N > 1: each rank copies
    # its input slab in, runs its step and copies its output band out; max over ranks.
    e2e = None
    if not args.no_e2e:
        fh = f_host.pin_memory()
        ohs = [torch.empty(tuple(out.shape), dtype=torch.float32).pin_memory() for _ in range(2)]
        n_e2e = max(1, min(args.steps, 3 if f.numel() * 4 > 256e6 else args.steps))

        # N = 1: frames through bf_vec_filter_host_async (H2D of frame i+1 and D2H of frame i-1
        # overlap frame i's kernels; every step still copies its input in and its result out),
        # one bf_vec_host_sync at the end; N > 1: per-rank copies around the sharded step
        def e2e_step(i):
            if world == 1:
                plan.filter_host_async(fh, ohs[i % 2])
            else:
                f.copy_(fh, non_blocking=True)
                step()
                ohs[0].copy_(out, non_blocking=True)
                torch.cuda.synchronize()

        def e2e_done():
            if world == 1:
                plan.host_sync()

        e2e_step(0)
        e2e_done()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n_e2e):
            e2e_step(i)
        e2e_done()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": cfg.H * cfg.W * cfg.M * n_e2e / float(e2e_s.item()), "unit": "pixel*samples/s",
               "h2d_bytes_per_step": fh.numel() * 4, "d2h_bytes_per_step": ohs[0].numel() * 4,
               "steps": n_e2e, "per_rank_bytes": world > 1,
               "api": "bf_vec_filter_host_async + bf_vec_host_sync (pipelined frames)" if world == 1
               else "per-rank H2D + sharded step + D2H"}

    clocks = clk.summary()
    pk = peaks()
    mhz_max = clocks.get("sm_max_mhz") or pk.get("sm_max_mhz") or 1965.0
    peak = fp32_peak_tflops(mhz_max)
    fused_ms = fused_ns / 1e6 / max(1, fused_calls)
    units_per_launch = rows * cfg.W * (k1 - k0)
    flops = (algorithmic_flops_per_px_sample(cfg.d, r) if args.engine == 0
             else recursive_flops_per_px_sample(cfg.d)) * units_per_launch
    achieved = flops / (fused_ms / 1e3) / 1e12
    kname = KERNEL_NAMES.get(plan.info("variant"), "mcsf_fused_kernel")
    if args.engine == 1:
        kname = {1: "rect_tile_kernel x3 + rect_scan_kernel x2",
                 2: "rect_tile_kernel x2 + rect_scan_kernel + rect_vscan_kernel"}.get(
                     plan.info("rec_impl"), "rec_row_kernel+rec_col_kernel")
        if plan.info("rec_impl") == 2 and plan.info("rec_tc") and plan.info("rec_vtc") and cfg.d == 3 \
                and cfg.W % 32 == 0:
            kname = kname.replace("rect_vscan_kernel", "rect_vscan_tc_kernel")
        if plan.info("rec_impl") >= 1 and plan.info("rec_tc") and cfg.d == 3:
            kname = kname.replace("rect_tile_kernel x2", "rect_tile_kernel + rect_tc2_kernel")
            kname = kname.replace("rect_tile_kernel x3", "rect_tile_kernel x2 + rect_tc2_kernel")
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": measured_traffic(cfg, kname, units_per_launch,
                                        {"tile_rows": plan.info("tile_rows"), "groups": plan.info("groups"),
                                         "persistent": plan.info("last_persistent")}),
            # algorithmic bytes per launch: read f, write S (8 d B per output pixel)
            "algorithmic_bytes": 8 * cfg.d * rows * cfg.W,
            "kernel": kname, "fused_ms_per_launch": fused_ms,
            "peak_source": f"FP32 pipe: 148 SM x 128 lanes x 2 flop x {mhz_max} MHz (sm_max)",
            "frac_at_run_clock": (achieved / fp32_peak_tflops(clocks["sm_mhz"])) if clocks.get("sm_mhz") else None,
            "flops_per_px_sample": (algorithmic_flops_per_px_sample(cfg.d, r) if args.engine == 0
                                    else recursive_flops_per_px_sample(cfg.d)),
            "fused_share_of_step": (fused_ns / 1e6) / ms if ms > 0 else None}
    roof["traffic_ratio"] = (roof["traffic"] / roof["algorithmic_bytes"]) if roof["traffic"] else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        bands_s, samples_s = cpu_sample_size(cfg)
        v, info = oracle_sample(cfg, bands_s, samples_s)
        cpu = cpu_baseline_entry(cfg, v, info, bands_s)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "pixel*samples/s", "n_gpus": world,
            "world_size": world, "communicator": comm,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(cfg, world, args.mode, l2=l2_note, tile_rows=plan.info("tile_rows"),
                                  engine=("recursive" if args.engine == 1 else "fir"),
                                  groups=plan.info("groups"), persistent=plan.info("last_persistent")),
            "mpix_per_s": cfg.H * cfg.W * args.steps / (ms_max / 1e3) / 1e6,
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def communicator_report(dist, dev, world):
    """One NCCL all_gather of each rank's (rank, local rank, PCI bus id): proves the communicator
    spans `world` distinct GPUs before anything is timed."""
    import torch
    props = torch.cuda.get_device_properties(dev)
    bus = int(getattr(props, "pci_bus_id", -1))
    mine = torch.tensor([dist.get_rank(), dev.index, bus], dtype=torch.int64, device=dev)
    got = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(got, mine)
    rows = [t.tolist() for t in got]
    ndev = len({(r[1], r[2]) for r in rows})
    rep = {"backend": dist.get_backend(), "nranks": dist.get_world_size(), "distinct_gpus": ndev,
           "ranks": [{"rank": r[0], "local_rank": r[1], "pci_bus_id": r[2]} for r in rows]}
    print(f"[rank {dist.get_rank()}] NCCL communicator: {dist.get_world_size()} ranks, "
          f"{ndev} distinct GPUs", file=sys.stderr, flush=True)
    return rep


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_command(argv, gpus, port):
    """The torchrun command bench.py re-executes itself under for --gpus N > 1 when it was not
    started by a launcher (one process per GPU, rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        import subprocess
        sys.exit(subprocess.call(launch_command(argv, args.gpus, free_port())))
    if world and world != args.gpus:
        if "--gpus" in " ".join(argv):
            sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks")
        args.gpus = world                      # torchrun without --gpus: the launcher's world
    from workloads import CONFIGS
    cfg = CONFIGS[args.config]
    if args.sigma:
        import dataclasses
        cfg = dataclasses.replace(cfg, sigma_s=args.sigma)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()

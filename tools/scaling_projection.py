"""Per-rank work of the multi-GPU partitions, timed on ONE GPU: what each of N ranks
runs in `bench.py --gpus N` for config 5, without the exchange. Sample shards: the full image with
M/N samples (bf_vec_filter_partial over [k0, k1)); row bands: an H/N-row band with its r-row halo
(bf_vec_filter_rows). Prints the projected compute-only efficiency T(N=1) / (N * T_rank(N))."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1605_02164_b200 import Plan, shard  # noqa: E402
from workloads import CONFIGS, make_image_rows  # noqa: E402

cfg = CONFIGS[5]
f = torch.from_numpy(make_image_rows(cfg, 0, cfg.H)).cuda()
s = torch.cuda.Stream()


def timed(fn, reps=3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(s):
        fn()
        s.synchronize()
        ts = []
        for _ in range(reps):
            ev[0].record(s)
            fn()
            ev[1].record(s)
            s.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
    return statistics.median(ts)


p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed)
p.sample_freqs()
out = torch.empty_like(f)
t1 = timed(lambda: p.filter(f, out))
print(f"N=1: {t1:.1f} ms")
for n in (2, 4, 8):
    k0, k1 = shard.sample_range(cfg.M, n, 0)
    PZ = torch.empty((cfg.d + 1) * cfg.H * cfg.W, device="cuda")
    ts = timed(lambda: p.filter_partial(f, k0, k1, PZ=PZ))
    y0, y1 = shard.band(cfg.H, n, 0)
    s0, s1 = shard.slab_for_band(cfg.H, cfg.radius, y0, y1)
    slab = f[:, s0:s1].contiguous()
    ob = torch.empty((cfg.d, y1 - y0, cfg.W), device="cuda")
    tb = timed(lambda: p.filter_rows(slab, s0, y0, y1, out=ob))
    print(f"N={n}: sample shard {ts:.1f} ms (compute-only efficiency {t1 / (n * ts):.3f}), "
          f"row band {tb:.1f} ms ({t1 / (n * tb):.3f})", flush=True)

"""Throughput of bf_vec_filter_batch on small images (config 1 and 2 shapes) vs one image per call."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402

for ci, nimg in ((1, 256), (2, 8)):
    cfg = CONFIGS[ci]
    f1 = torch.from_numpy(make_image(cfg)).cuda()
    fb = f1.unsqueeze(0).repeat(nimg, 1, 1, 1).contiguous()
    out = torch.empty_like(fb)
    p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed)
    p.sample_freqs()
    s = torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(s):
        for label, fn in (("single", lambda: p.filter(f1, out[0])), ("batch", lambda: p.filter_batch(fb, out))):
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.3:
                fn()
                s.synchronize()
            ts = []
            for _ in range(9):
                ev[0].record(s)
                fn()
                ev[1].record(s)
                s.synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
            ms = statistics.median(ts)
            n = nimg if label == "batch" else 1
            print(f"config {ci} {label} x{n}: {ms:.3f} ms, {n * cfg.H * cfg.W * cfg.M / ms * 1e3:.4e} px*samples/s",
                  flush=True)

"""Time bf_vec_filter with Gaussian / box / hat spatial taps on configs 5, 3, 2 (same images, M)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402

for ci in (5, 3, 2):
    cfg = CONFIGS[ci]
    f = torch.from_numpy(make_image(cfg)).cuda()
    out = torch.empty_like(f)
    s = torch.cuda.Stream()
    for kind in (0, 1, 2):
        p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed)
        p.set_option("spatial_kernel", kind)
        p.sample_freqs()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.5:
                p.filter(f, out)
                s.synchronize()
            ts = []
            for _ in range(5):
                ev[0].record(s)
                p.filter(f, out)
                ev[1].record(s)
                s.synchronize()
                ts.append(ev[0].elapsed_time(ev[1]))
        ms = statistics.median(ts)
        print(f"config {ci} spatial {kind} variant {p.info('variant')}: {ms:.3f} ms "
              f"{cfg.H * cfg.W * cfg.M / ms * 1e3:.4e} px*samples/s", flush=True)
        p.close()

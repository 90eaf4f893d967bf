"""Minimal Python user of the binding: filter a synthetic image on the GPU with the default
(fused FIR) engine and with the recursive O(1) engine, and compare both with the exact filter.

    python examples/filter_torch.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402

cfg = CONFIGS[2]                                              # 512 x 512 RGB, sigma_s = 5, M = 64
f = torch.from_numpy(make_image(cfg)).cuda()
with Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed) as p:
    p.sample_freqs()
    exact = p.direct(f)                                       # Eq. (2)-(3), O(r^2) per pixel
    for engine in (0, 1):
        p.set_option("engine", engine)
        S = p.filter(f)                                       # Algorithm 1 (MCSF)
        zmin, nsmall = p.diag()
        Z = p.filter_partial(f, 0, cfg.M).reshape(cfg.d + 1, cfg.H, cfg.W)[cfg.d]
        ok = Z / cfg.M >= 0.05                                # pixels whose MC denominator is conditioned
        err = (S.double() - exact.double()) ** 2
        psnr = lambda e: 10 * np.log10(255.0 ** 2 / e.mean().item())  # noqa: E731
        print(f"engine {engine}: PSNR vs exact {psnr(err):.1f} dB over all pixels, "
              f"{psnr(err[:, ok]):.1f} dB over the {int(ok.sum())} with Z/M >= 0.05 "
              f"(min Z/M {zmin:.3f}, {nsmall} below)")

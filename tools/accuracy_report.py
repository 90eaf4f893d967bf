"""Accuracy of the MC filter against the exact direct filter (Eq. (20)),
both computed by libbfvec on the GPU, per BASELINE config: MSE, the paper's
"MSE dB" = 10 log10(MSE) (reading R13), PSNR = 10 log10(R^2/MSE), over all pixels and
over pixels with Z/M >= 0.05 (reading R5). Prints one JSON line per config."""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3,4,5")
args = ap.parse_args()
for i in [int(c) for c in args.configs.split(",")]:
    cfg = CONFIGS[i]
    f = torch.from_numpy(make_image(cfg)).cuda()
    p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed, value_range=cfg.value_range)
    p.sample_freqs()
    S = p.filter(f)
    zmin, nsmall = p.diag()
    Z = p.filter_partial(f, 0, cfg.M).reshape(cfg.d + 1, cfg.H, cfg.W)[cfg.d]
    B = p.direct(f)
    torch.cuda.synchronize()
    err = (S.double() - B.double()) ** 2
    ok = (Z / cfg.M >= 0.05)
    mse_all = float(err.mean())
    mse_ok = float(err[:, ok].mean())
    R = cfg.value_range
    line = {"config": cfg.name, "mse": mse_all, "mse_db": 10 * math.log10(mse_all),
            "psnr_db": 10 * math.log10(R * R / mse_all), "mse_conditioned": mse_ok,
            "psnr_conditioned_db": 10 * math.log10(R * R / mse_ok), "excluded_px": int((~ok).sum()),
            "z_min_over_M": zmin, "n_small_z": nsmall}
    print(json.dumps(line), flush=True)
    del f, S, Z, B
    p.close()
    torch.cuda.empty_cache()

"""Times the exact filter (bf_vec_direct, csrc/direct.cu) against its roofline.

    python tools/direct_bench.py [--reps 10] [--json out.json]

Rows: the paper's Table 1 (512x512 colour image, sigma_r = 40, sigma_s = 1..10;
here the config-2 stand-in image) and BASELINE configs 2-5 at their own sigma_s.

Algorithmic work per (output pixel, window offset) pair: 3d + 1 FP32 lane-ops (d differences,
d FFMA for the quadratic form, d FFMA + 1 FADD for the weighted sums; the log2 spatial weight
is the FFMA chain's addend) and 1 MUFU.EX2. Roofline: the slower of the FP32 pipe
(148 SM x 128 lanes x clock) and the MUFU pipe (148 SM x 16 / clk x clock).
"""
import argparse
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402

MHZ = 1965.0


def bound_s(pairs, d, mhz=MHZ):
    fp32 = pairs * (3 * d + 1) / (148 * 128 * mhz * 1e6)
    mufu = pairs / (148 * 16 * mhz * 1e6)
    return max(fp32, mufu), ("fp32" if fp32 >= mufu else "mufu")


def time_direct(cfg, f, reps, rows=0):
    p = Plan(cfg.H, cfg.W, cfg.d, cfg.sigma_s, cfg.C_array, cfg.N, cfg.M, cfg.seed, value_range=cfg.value_range)
    p.set_option("direct_rows", rows)
    out = torch.empty_like(f)
    s = torch.cuda.current_stream()
    for _ in range(3):
        p.direct(f, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        p.direct(f, out)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    p.close()
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--json", default="")
    ap.add_argument("--only", default="", help="run only cases whose name contains this")
    ap.add_argument("--rows", type=int, default=0, help="option direct_rows (0 auto, 4, 8, 16)")
    args = ap.parse_args()
    rows = []
    c2 = CONFIGS[2]
    f2 = torch.from_numpy(make_image(c2)).cuda()
    cases = [(f"table1_sigma{s}", dataclasses.replace(c2, sigma_s=float(s), C=((1600.0, 0, 0), (0, 1600.0, 0),
                                                                              (0, 0, 1600.0))), f2)
             for s in (1, 2, 3, 4, 5, 10)]
    for i in (2, 3, 4, 5):
        cfg = CONFIGS[i]
        cases.append((cfg.name, cfg, None))
    for name, cfg, f in cases:
        if args.only and args.only not in name:
            continue
        if f is None:
            f = torch.from_numpy(make_image(cfg)).cuda()
        ms = time_direct(cfg, f, args.reps, args.rows)
        r = cfg.radius
        pairs = cfg.H * cfg.W * (2 * r + 1) ** 2
        b, which = bound_s(pairs, cfg.d)
        row = {"case": name, "direct_rows": args.rows, "H": cfg.H, "W": cfg.W, "d": cfg.d, "sigma_s": cfg.sigma_s, "r": r, "ms": ms,
               "pairs_per_s": pairs / (ms / 1e3), "bound_ms": b * 1e3, "bound": which,
               "frac_of_roofline": b * 1e3 / ms}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del f
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()

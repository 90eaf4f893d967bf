"""Small launches of every kernel family for compute-sanitizer.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [--case NAME ...]

Each case builds a plan on a small synthetic image, runs it once through the C ABI
(CUDA graphs off, so every kernel is a plain launch the sanitizer instruments), and
checks the raw sums against the C oracle's Algorithm 1 (Gate A) so a run that is
clean but wrong is caught too. Sizes are chosen so each case finishes in seconds under
racecheck (which serialises shared-memory accesses).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# name -> (d, H, W, sigma_s, M, options)
CASES = {
    "v6_r6": (3, 40, 72, 2.0, 4, {}),            # CfgT2<3,6>   (config 1's radius)
    "v6_r15": (3, 48, 80, 5.0, 4, {}),           # CfgT2<3,15>  (config 2's radius)
    "v6_r48": (3, 24, 40, 16.0, 2, {}),          # CfgT2<3,48>  (config 5's radius, multi-fold reflection)
    "v8_d8": (8, 40, 72, 2.0, 3, {}),            # variant 8 (two launches, programmatic dependent launch)
    "box_r15": (3, 48, 80, 5.0, 4, {"spatial_kernel": 1}),   # running-sum instance
    "rec_tiled": (3, 40, 72, 2.0, 3, {"engine": 1, "rec_impl": 1}),
    "rec_staged": (3, 40, 72, 2.0, 3, {"engine": 1, "rec_impl": 0}),
    "direct": (3, 40, 72, 2.0, 2, {"direct": 1}),
}


def run_case(name):
    import torch

    from oracle import draws, native
    from oracle import plan as oplan
    from paper_1605_02164_b200 import Plan
    from workloads.configs import random_image

    d, H, W, sigma, M, opts = CASES[name]
    opts = dict(opts)
    C = np.eye(d) * (40.0 ** 2 if d != 8 else 0.3 ** 2)
    vr = 255.0 if d != 8 else 1.0
    f = random_image(H, W, d, seed=7, value_range=vr, smooth=True)
    p = Plan(H, W, d, sigma, C, 20, M, 5, value_range=vr)
    p.set_option("graph", 0)
    direct = opts.pop("direct", 0)
    for k, v in opts.items():
        p.set_option(k, v)
    p.sample_freqs()
    fg = torch.from_numpy(f).cuda()
    if direct:
        out = p.direct(fg).cpu().numpy()
        ref = native.direct_full(f, C, sigma)
        err = np.abs(out - ref).max() / vr
        print(f"{name}: direct max err {err:.2e}")
        assert err <= 1e-3
        return
    out = p.filter(fg)
    PZ = p.filter_partial(fg, 0, M).cpu().numpy().reshape(d + 1, H, W)
    torch.cuda.synchronize()
    Q, a = oplan.diagonalize(C)
    Y = draws.y_draws(5, M, d, 20)
    spatial = {1: "box"}.get(opts.get("spatial_kernel", 0), "gaussian")
    if opts.get("engine", 0) == 1:
        spatial = "deriche"
    _, P, Z = native.mcsf_full(f, Q, a, 20, Y, sigma, spatial=spatial)
    gate = max(np.abs(PZ[d] - Z).max() / M, np.abs(PZ[:d] - P).max() / M / vr)
    print(f"{name}: variant {p.info('variant')} engine {p.info('engine')} gate A {gate:.2e}; "
          f"out finite {bool(torch.isfinite(out).all())}")
    assert gate <= 1e-5
    p.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", nargs="*", default=list(CASES))
    args = ap.parse_args()
    for c in args.case:
        run_case(c)
    print("sanitize_run: all cases done")


if __name__ == "__main__":
    main()

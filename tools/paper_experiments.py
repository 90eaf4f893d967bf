"""The paper's two experiments re-run on B200 with the library (synthetic stand-ins):

  table1  Table 1: run time vs sigma_s on a 512 x 512 colour image,
          sigma_r = 40, N = 10, T = 300, for the exact direct filter (bf_vec_direct), the MC filter
          with the truncated FIR (engine 0) and with the recursive O(1) engine (engine 1).
  fig5    Fig. 5: Eq. (20) MSE between the exact filter and MCSF vs T, averaged
          over R realisations, sigma_s = 1, sigma_r = 30, N in {10, 20} (bf_vec_mse_sweep), iid and
          stratified draws.

The paper used the Peppers / Dome photographs; the 512 x 512 Voronoi image of config 2 stands in
(same size as Peppers). Prints one JSON object per experiment row; --out writes them all.
"""
import argparse
import json
import math
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1605_02164_b200 import Plan  # noqa: E402
from workloads import CONFIGS, make_image  # noqa: E402


def timed(fn, reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:          # clock ramp-up
        fn()
        torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return statistics.median(ts)


def table1(f, rows, reps):
    d = f.shape[0]
    C = np.eye(d) * 40.0 ** 2
    for s in (1, 2, 3, 4, 5, 10):
        row = {"experiment": "table1", "sigma_s": s, "sigma_r": 40, "N": 10, "T": 300, "H": f.shape[1],
               "W": f.shape[2]}
        for eng in (0, 1):
            p = Plan(f.shape[1], f.shape[2], d, float(s), C, 10, 300, 1)
            p.set_option("engine", eng)
            p.sample_freqs()
            out = torch.empty_like(f)
            row["mcsf_fir_ms" if eng == 0 else "mcsf_recursive_ms"] = timed(lambda: p.filter(f, out), reps)
            p.close()
        p = Plan(f.shape[1], f.shape[2], d, float(s), C, 10, 300, 1)
        out = torch.empty_like(f)
        row["direct_ms"] = timed(lambda: p.direct(f, out), reps)
        p.close()
        print(json.dumps(row), flush=True)
        rows.append(row)


def fig5(f, rows, nreal, t_list):
    d = f.shape[0]
    C = np.eye(d) * 30.0 ** 2
    ref_plan = Plan(f.shape[1], f.shape[2], d, 1.0, C, 10, max(t_list), 0)
    ref = ref_plan.direct(f)
    for sampler in ("iid", "stratified"):
        for N in (10, 20):
            p = Plan(f.shape[1], f.shape[2], d, 1.0, C, N, max(t_list), 0)
            p.set_option("sampler", 0 if sampler == "iid" else 1)
            p.sample_freqs()
            t0 = time.perf_counter()
            mse = p.mse_sweep(f, ref, list(range(1000, 1000 + nreal)), t_list)
            secs = time.perf_counter() - t0
            mean = mse.mean(axis=0)
            row = {"experiment": "fig5", "sampler": sampler, "N": N, "sigma_s": 1, "sigma_r": 30,
                   "realisations": nreal, "T": t_list, "mse_mean": mean.tolist(),
                   "mse_db": [10 * math.log10(m) for m in mean],
                   "mse_sem": (mse.std(axis=0, ddof=1) / math.sqrt(nreal)).tolist(), "seconds": secs}
            print(json.dumps(row), flush=True)
            rows.append(row)
            p.close()


def lab_bandwidth(rows, reps):
    """sRGB <-> CIE-Lab transforms on the 8192^2 config-5 image: HBM-bound,
    12 B read + 12 B written per pixel; reported against the measured copy bandwidth."""
    from paper_1605_02164_b200 import lab_to_srgb, srgb_to_lab
    f = torch.from_numpy(make_image(CONFIGS[5])).cuda()
    out = torch.empty_like(f)
    npix = f.shape[1] * f.shape[2]
    peak = None
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as fh:
            peak = json.load(fh).get("hbm_gbs")
    except Exception:
        pass
    for name, fn in (("srgb_to_lab", lambda: srgb_to_lab(f, out=out)), ("lab_to_srgb", lambda: lab_to_srgb(f, out=out))):
        ms = timed(fn, reps)
        gbs = 24.0 * npix / (ms / 1e3) / 1e9
        row = {"experiment": "lab", "kernel": name, "pixels": npix, "ms": ms, "GB_per_s": gbs,
               "hbm_peak_GB_per_s": peak, "frac": (gbs / peak) if peak else None}
        print(json.dumps(row), flush=True)
        rows.append(row)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="table1,fig5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--realisations", type=int, default=400)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    f = torch.from_numpy(make_image(CONFIGS[2])).cuda()
    rows = []
    if "table1" in a.which:
        table1(f, rows, a.reps)
    if "fig5" in a.which:
        fig5(f, rows, a.realisations, [25, 50, 100, 200, 300, 400])
    if "lab" in a.which:
        lab_bandwidth(rows, a.reps)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()

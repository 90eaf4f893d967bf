"""Checks bench.py's halo-corrected CPU extrapolation against a full-image oracle run.

    python tools/cpu_halo_check.py [--config 3] [--samples 4]

Times Algorithm 1 (oracle, fp64 OpenMP, all host cores) on the whole image of a config that
fits in seconds, and on three bands of 64 / 128 / 256 rows of the same image, and prints the
measured band throughput, the halo factor and the ratio full / (measured x halo factor).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--samples", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    full = max(bench.oracle_sample(cfg, [(0, cfg.H)], a.samples)[0] for _ in range(a.reps))
    print(f"{cfg.name}: full image {full:.4g} px*samples/s (best of {a.reps})")
    for rows in (64, 128, 256):
        mid = cfg.H // 2 - rows // 2
        bands = [(0, rows), (mid, mid + rows), (cfg.H - rows, cfg.H)]
        v = max(bench.oracle_sample(cfg, bands, a.samples)[0] for _ in range(a.reps))
        hf = bench.halo_factor(cfg, bands)
        print(f"  {rows}-row bands: measured {v:.4g}, halo factor {hf:.3f}, estimate {v * hf:.4g}, "
              f"full / estimate {full / (v * hf):.3f}")


if __name__ == "__main__":
    main()

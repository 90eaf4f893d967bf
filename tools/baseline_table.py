"""Render BASELINE.md §4 ("Measured") from the committed bench lines.

    python tools/baseline_table.py profiles/r02_bench_c{1,2,3,4,5}.json

One row per bench line (bench.py on one B200): SM clock under load, fused-kernel ms (CUDA events
on the launching stream), whole-step ms, end-to-end ms per frame (pipelined host frames),
pixel*samples/s, MPix/s, the FP32-pipe fraction (the roofline), the MUFU and HBM
fractions of the same run (2 MUFU per pixel-sample at 16/clk/SM; 8 d algorithmic bytes per pixel
against MEASURED_PEAKS.json hbm_gbs), and the CPU oracle's throughput with its core count.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(paths):
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"] * 1e9
    print("| cfg | GPUs | schedule | SM clock (MHz) | kernel ms | step ms | e2e ms / frame | px·samples/s | MPix/s "
          "| % FP32 roofline | % SFU | % HBM | e2e / device | CPU oracle px·samples/s (cores) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        d = json.loads(open(p).read().strip().splitlines()[-1])
        c, r = d["config"], d["roofline"]
        mhz = d["clocks"]["sm_mhz"] or 1965.0
        units = c["H"] * c["W"] * c["M"]
        t = d["ms_per_step"] / 1e3
        mufu = 2 * d["value"] / (148 * 16 * mhz * 1e6)
        hbm_frac = 8 * c["d"] * c["H"] * c["W"] / t / hbm
        e2e = d.get("e2e") or {}
        e2e_ms = units / e2e["value"] * 1e3 if e2e.get("value") else None
        cpu = d.get("cpu_baseline") or {}
        sched = ("persistent" if c.get("persistent") else f"{c.get('tile_rows')} rows") + f", {c.get('groups')} slots"
        cpu_s = (f"{cpu['value']:.3g} ({cpu['cores']}{', extrap.' if cpu.get('extrapolated') else ''})"
                 if cpu.get("value") else "—")
        print(f"| {c['workload']} | {d['n_gpus']} | {sched} | {mhz:.0f} | {r['fused_ms_per_launch']:.4g} "
              f"| {d['ms_per_step']:.4g} | {e2e_ms:.4g} | {d['value']:.4g} | {d['mpix_per_s']:.4g} "
              f"| {100 * r['frac']:.1f} | {100 * mufu:.2f} | {100 * hbm_frac:.3f} "
              f"| {e2e['value'] / d['value']:.3f} | {cpu_s} |")


if __name__ == "__main__":
    main(sys.argv[1:])

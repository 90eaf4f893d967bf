"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: markdown table."""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    k = r[ix["Kernel Name"]].split("(")[0][:80]
    agg[k][0] += 1
    agg[k][1] += float(r[ix["Metric Value"]].replace(",", "")) * SCALE[r[ix["Metric Unit"]]]
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | total | share of GPU time |\n|---|---|---|---|")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {ms:.2f} ms | {100 * ms / tot:.2f} % |")

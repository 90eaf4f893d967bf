"""Summarise an ncu report (details + stall attribution per SASS region) for profiles/."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


keys = ["Duration", "SM Frequency", "Registers Per Thread", "Achieved Occupancy", "Issue Slots Busy",
        "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Executed Instructions", "DRAM Throughput", "L2 Hit Rate", "Dynamic Shared Memory Per Block",
        "Compute (SM) Throughput", "Memory Throughput", "No Eligible"]
rows = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keys:
        print(f"{d['Metric Name']:45s} {d['Metric Value']:>16s} {d['Metric Unit']}")
    if d.get("Metric Name", "").startswith("INF") or "pipeline" in d.get("Rule Description", ""):
        pass
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
for h, u, v in zip(raw[0], raw[1], raw[2]):
    if ("pipe_fma" in h or "pipe_fp" in h or "pipe_xu" in h or "pipe_lsu" in h or "inst_executed_pipe_fmaheavy" in h
            or "dram__bytes_read.sum" == h or "dram__bytes_write.sum" == h) and ("pct" in h or "bytes" in h):
        print(f"{h:70s} {v:>14s} {u}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv"))))
shdr = src[1]
ix = {h: i for i, h in enumerate(shdr)}
data = src[2:]
tot = sum(int(r[ix["# Samples"]]) for r in data) or 1
byop = collections.Counter()
stall_cols = [h for h in shdr if h.startswith("stall_") and "Not Issued" not in h]
stalls = collections.Counter()
for r in data:
    toks = r[ix["Source"]].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    byop[op.split(".")[0]] += int(r[ix["# Samples"]])
    for h in stall_cols:
        try:
            stalls[h] += int(r[ix[h]])
        except ValueError:
            pass
print("\nPC samples by opcode:")
for op, c in byop.most_common(12):
    print(f"  {op:10s} {100 * c / tot:5.1f} %")
print("stall reasons (all samples):")
for h, c in stalls.most_common(10):
    print(f"  {h:25s} {100 * c / tot:5.1f} %")

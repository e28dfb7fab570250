"""Summarise an ncu report: key SOL metrics + top source lines by stall samples.
Usage: python profiles/ncu_summary.py report.ncu-rep [top_n] [file:lo-hi=region ...]
NCU_LAUNCH=i selects the i-th profiled launch of a multi-launch report."""
import collections
import csv
import io
import subprocess
import os
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def run(*a):
    sel = ["--launch-skip", os.environ["NCU_LAUNCH"], "--launch-count", "1"] if "NCU_LAUNCH" in os.environ else []
    return subprocess.run(["ncu", "-i", rep, *sel, *a], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
want = {"Duration", "DRAM Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Warp Cycles Per Issued Instruction", "No Eligible", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size", "Memory Throughput", "Avg. Active Threads Per Warp"}
for r in det[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:38s} {d['Metric Value']} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
d = dict(zip(raw[0], raw[2] if len(raw) > 2 else raw[1]))
for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "gpu__time_duration.sum"):
    print(k, d.get(k), raw[1][raw[0].index(k)] if k in raw[0] else "")
stalls = {k: v for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
for k, v in sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]:
    print("  stall", k.replace("smsp__pcsamp_warps_issue_stalled_", ""), v)
rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source=cuda,sass"))))
res, inst, text = collections.Counter(), collections.Counter(), {}
fname, hdr = None, None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    dd = dict(zip(hdr, r))
    try:
        res[(fname, ln)] += float(dd.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst[(fname, ln)] += float(dd.get("Instructions Executed", "0") or 0)
    except ValueError:
        pass
    text[(fname, ln)] = r[1].strip()[:80]
ts, ti = sum(res.values()) or 1, sum(inst.values()) or 1
print(f"source lines (samples {ts:.0f}, instructions {ti:.0f})")
for k, v in res.most_common(top):
    print(f"  {k[0]}:{k[1]:<5d} samp {100 * v / ts:5.1f}%  inst {100 * inst[k] / ti:5.1f}%  {text[k]}")

# optional region aggregation: pass "file:lo-hi=name" specs after top_n
specs = sys.argv[3:]
if specs:
    agg_s, agg_i = collections.Counter(), collections.Counter()
    for (f, ln), v in res.items():
        name = "other"
        for sp in specs:
            rng, nm = sp.split("=")
            ff, lr = rng.split(":")
            lo, hi = (int(x) for x in lr.split("-"))
            if f == ff and lo <= ln <= hi:
                name = nm
                break
        agg_s[name] += v
        agg_i[name] += inst[(f, ln)]
    for (f, ln), v in inst.items():
        if (f, ln) not in res:
            pass
    print("regions:")
    for nm in sorted(agg_i, key=lambda k: -agg_i[k]):
        print(f"  {nm:20s} samples {100 * agg_s[nm] / ts:5.1f}%  instructions {100 * agg_i[nm] / ti:5.1f}%")

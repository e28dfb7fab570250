"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launches / total time / share. Usage: launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
cnt, tot = collections.Counter(), collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("msim_impl::", "").replace("(anonymous namespace)::", "")
    cnt[name] += 1
    tot[name] += float(r[vi].replace(",", ""))
all_t = sum(tot.values()) or 1.0
print(f"# {'kernel':44s} {'launches':>8s} {'total_ns':>14s}  share")
for k, v in tot.most_common():
    print(f"  {k[-44:]:44s} {cnt[k]:8d} {v:14.1f}  {100 * v / all_t:5.2f}%")

"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file X.csv): time per kernel name, count and share.
    python tools/launch_table.py X.csv"""
import collections
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    k = r[ki].split("(")[0].replace("<unnamed>::", "").replace("void ", "")[:60]
    agg.setdefault(k, [0, 0.0])
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}% {c:5d}x  {k}")
print(f"{tot / 1e3:10.1f} us total, {sum(v[0] for v in agg.values())} launches")

"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    v *= scale.get(r[ui], 1e-3)
    agg[r[ki].split("(")[0]].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':58s} {'n':>5s} {'mean_us':>12s} {'total_us':>12s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:58]:58s} {len(v):5d} {sum(v)/len(v):12.2f} {sum(v):12.1f} {sum(v)/tot:6.1%}")

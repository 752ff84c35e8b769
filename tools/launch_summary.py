"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel count, total and share.  python tools/launch_summary.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"{'us':>12} {'share':>6} {'n':>6}  kernel")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:12.1f} {100 * v / tot:5.1f}% {c:6d}  {k[:100]}")
print(f"total {tot / 1e3:.3f} ms over {sum(c for c, _ in agg.values())} launches")

"""Summarise an ncu --csv launch list (gpu__time_duration.sum and, when
captured, dram__bytes_read.sum / dram__bytes_write.sum): per-kernel count,
total time, share, DRAM bytes per launch.

    python tools/launch_summary.py file.csv [--json out.json]"""
import collections
import csv
import json
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui, mi = (h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"),
                  h.index("Metric Name"))
idi = h.index("ID")
tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
          "second": 1e6, "s": 1e6}
bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
          "GB": 1e9, "B": 1.0}
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    key = r[idi]
    name = r[ki].split("(")[0].replace("void ", "")
    rec = launch.setdefault(key, {"name": name, "us": 0.0, "dram": 0.0})
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        rec["us"] = v * tscale.get(r[ui], 1.0)
    elif r[mi].startswith("dram__bytes"):
        rec["dram"] += v * bscale.get(r[ui], 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for rec in launch.values():
    a = agg[rec["name"]]
    a[0] += 1
    a[1] += rec["us"]
    a[2] += rec["dram"]
tot = sum(a[1] for a in agg.values())
print(f"{'us':>12} {'share':>6} {'n':>6} {'MB/launch':>10}  kernel")
for k, (c, v, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:12.1f} {100 * v / tot:5.1f}% {c:6d} {b / c / 1e6:10.2f}  {k[:100]}")
print(f"total {tot / 1e3:.3f} ms over {len(launch)} launches")
if "--json" in sys.argv:
    out = {k: {"launches": c, "us": v, "dram_bytes": b} for k, (c, v, b) in agg.items()}
    json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)

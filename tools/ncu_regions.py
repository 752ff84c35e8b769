"""Per-region stall breakdown of an ncu source page (SASS), splitting the
kernel at barrier / mbarrier instructions.  python tools/ncu_regions.py rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
isrc = h.index("Source")
iex = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ir = [h.index(c) for c in reasons]
tot = sum(float(r[h.index("Warp Stall Sampling (All Samples)")] or 0) for r in data)
regions, cur = [], {"start": 0, "ops": 0, "s": [0.0] * len(ir), "label": ""}
for i, r in enumerate(data):
    src = r[isrc].strip()
    ex = float(r[iex] or 0)
    for k, j in enumerate(ir):
        cur["s"][k] += float(r[j] or 0)
    if ex > 0:
        cur["ops"] += ex
    if "BAR.SYNC" in src or "SYNCS.PHASECHK" in src:
        cur["label"] = src[:40]
        cur["end"] = i
        regions.append(cur)
        cur = {"start": i + 1, "ops": 0, "s": [0.0] * len(ir), "label": ""}
cur["end"] = len(data)
cur["label"] = "(tail)"
regions.append(cur)
for g in regions:
    s = sum(g["s"])
    if s < 0.01 * tot:
        continue
    top = sorted(zip(g["s"], reasons), reverse=True)[:4]
    print(f"[{g['start']:5d}-{g['end']:5d}] {100 * s / tot:5.1f}% ends {g['label']:40s} " +
          " ".join(f"{n.replace('stall_', '')}={100 * v / tot:.1f}" for v, n in top))

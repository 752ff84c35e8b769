"""Top stall-sampled SASS lines of an ncu source-page CSV (--print-source sass),
with per-region totals.  python tools/sass_hot.py page.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ai, si, ti = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ni = h.index("Warp Stall Sampling (Not-issued Samples)")
ei = h.index("Instructions Executed")
recs = []
for r in rows[2:]:
    if len(r) <= ti:
        continue
    try:
        recs.append((int(r[ti]), int(r[ni]), int(r[ei] or 0), r[ai][-5:], r[si].strip()))
    except ValueError:
        pass
tot = sum(x[0] for x in recs)
print(f"total samples {tot}, instructions {sum(x[2] for x in recs)}")
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, nis, e, a, src in sorted(recs, reverse=True)[:N]:
    print(f"{100 * s / tot:5.2f}% ni={nis:6d} ex={e:9d} {a} {src[:90]}")
ops = {}
for s, nis, e, a, src in recs:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    o = ops.setdefault(op, [0, 0])
    o[0] += s
    o[1] += e
print("by opcode:", ", ".join(f"{k}={100 * v[0] / tot:.1f}%/{v[1]}" for k, v in
                            sorted(ops.items(), key=lambda x: -x[1][0])[:16]))

"""In-situ timeline of the 1-GPU cascade schedule: per block, how long the
panel (side stream) and the update (main stream) take while they overlap.

    python tools/cascade_profile.py [--m 2000 --n 20000] [--csv out.csv]

Drives the same building blocks the library's cascade uses (pdas_cascade_panel
/ pdas_cascade_update, side-stream lookahead) through dist.cascade_schedule with
one rank, recording CUDA events around every launch.  Inputs are synthetic
([Y | x] random, d = 10^U[-1,1]); the cost does not depend on the values."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200 import dist as D  # noqa: E402
from paper_1502_03543_b200._lib import load  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2000)
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--csv", default=None)
args = ap.parse_args()
m, n = args.m, args.n
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
cols0 = torch.rand(m * (n + 1), dtype=torch.float64, device="cuda", generator=g) * 1e-3
d = torch.pow(10.0, torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
cols = cols0.clone()
ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8, device="cuda")
fail = torch.zeros(1, dtype=torch.int32, device="cuda")


class Timed(D.CudaShard):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.ev = []

    def _rec(self, kind, b, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        e0.record(s)
        fn()
        e1.record(s)
        self.ev.append((kind, b, e0, e1))

    def panel(self, q0, p0, p1):
        self._rec("panel", p0 // self.plan.B, lambda: super(Timed, self).panel(q0, p0, p1))

    def update(self, p0, p1, i0):
        self._rec("update", p0 // self.plan.B, lambda: super(Timed, self).update(p0, p1, i0))


plan = D.make_plan(m, n, 1, 0)
for rep in range(2):
    cols.copy_(cols0)
    be = Timed(plan, cols, A, d, ws, fail, streams=True)
    be.epoch = rep * 10
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    D.run_lockstep([plan], [be])
    t1.record()
    torch.cuda.synchronize()
total = t0.elapsed_time(t1)
rows = []
for kind, b, e0, e1 in be.ev:
    rows.append((kind, b, t0.elapsed_time(e0), t0.elapsed_time(e1)))
P = {b: (s, e) for k, b, s, e in rows if k == "panel"}
U = {b: (s, e) for k, b, s, e in rows if k == "update"}
nb = plan.nb
# block b's step: from the end of update(b-1) to the end of update(b)
crit_panel = 0.0
print(f"m={m} n={n} blocks={nb} tile={plan.w} total {total:.2f} ms")
print(" b   panel(b+1) ms   update(b) ms   gap(b) ms")
prev_end = 0.0
waits = 0.0
for b in range(nb):
    pu = P.get(b + 1, (0, 0))
    uu = U.get(b, (prev_end, prev_end))
    gap = uu[0] - prev_end  # main stream idle waiting for panel(b)
    waits += max(gap, 0.0)
    if b % 10 == 0 or b >= nb - 5:
        print(f"{b:3d} {pu[1] - pu[0]:12.3f} {uu[1] - uu[0]:14.3f} {gap:11.3f}")
    prev_end = uu[1]
psum = sum(e - s for s, e in P.values())
usum = sum(e - s for s, e in U.values())
print(f"sum panel {psum:.1f} ms, sum update {usum:.1f} ms, main-stream waits on panels {waits:.1f} ms")
if args.csv:
    with open(args.csv, "w") as f:
        f.write("kind,block,start_ms,end_ms\n")
        for r in rows:
            f.write("%s,%d,%.4f,%.4f\n" % r)

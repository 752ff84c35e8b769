"""Per-block timeline of the library's own 1-GPU cascade (update on the main
stream, panel on the side stream), from CUDA events the library records when
PDAS_CASCADE_PROFILE=1.

    python tools/cascade_timeline.py [--m 2000 --n 20000]

Prints, every 10th block, the panel and update durations and how long the
main stream sat idle waiting for the panel, plus the totals."""
import argparse
import ctypes
import os
import sys

os.environ["PDAS_CASCADE_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200._lib import call, load  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2000)
ap.add_argument("--n", type=int, default=20000)
args = ap.parse_args()
m, n = args.m, args.n
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
cols0 = torch.rand(m * (n + 1), dtype=torch.float64, device="cuda", generator=g) * 1e-3
d = torch.pow(10.0, torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
cols = cols0.clone()
ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8, device="cuda")
fail = torch.zeros(1, dtype=torch.int32, device="cuda")
for rep in range(2):
    cols.copy_(cols0)
    call("pdas_solve_sweeps_ws", dv.ptr(cols), dv.ptr(A), dv.ptr(d), m, n, dv.ptr(ws), rep + 1,
         dv.ptr(fail), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
nr = int(load().pdas_debug_cascade_profile(None, 0))
buf = (ctypes.c_double * (4 * nr))()
load().pdas_debug_cascade_profile(ctypes.addressof(buf), nr)
rows = np.frombuffer(buf, dtype=np.float64).reshape(nr, 4)
U = {int(b): (s, e) for k, b, s, e in rows if k == 0}
P = {int(b): (s, e) for k, b, s, e in rows if k == 1}
nb = max(U) + 1
total = max(e for _, _, _, e in rows)
print(f"m={m} n={n} blocks={nb} cascade {total:.2f} ms")
print("  b  panel(b) ms  update(b) ms  main idle before U(b) ms")
idle = 0.0
prev = 0.0
for b in range(nb):
    ps, pe = P.get(b, (0.0, 0.0))
    us, ue = U[b]
    gap = max(us - prev, 0.0)
    idle += gap
    if b % 10 == 0 or b >= nb - 3:
        print(f"{b:4d} {pe - ps:11.3f} {ue - us:13.3f} {gap:12.3f}")
    prev = ue
print(f"sum panel {sum(e - s for s, e in P.values()):.1f} ms, sum update "
      f"{sum(e - s for s, e in U.values()):.1f} ms, main idle {idle:.1f} ms")

"""One panel hop on the timeline (a -DPDAS_HOP_TRACE=1 build): tile 15 of pivot
block 5 finishing and publishing its final columns, tile 16 seeing the flag,
staging the denominators and applying the published pivots.

    make -C paper_1502_03543_b200/csrc variant VDEFS=-DPDAS_HOP_TRACE=1 VNAME=hop
    PDAS_B200_LIB=paper_1502_03543_b200/csrc/build/var_hop/libpdas_b200.so \\
        python tools/hop_trace.py [--m 500 --n 5000]"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200._lib import call, load  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=500)
ap.add_argument("--n", type=int, default=5000)
ap.add_argument("--legacy", action="store_true",
                help="the CTA-wide panel's marks (k_casc_panel: m > 2048)")
args = ap.parse_args()
m, n = args.m, args.n
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
cols = torch.rand(m * (n + 1), dtype=torch.float64, device="cuda", generator=g) * 1e-3
d = torch.pow(10.0, torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8, device="cuda")
fail = torch.zeros(1, dtype=torch.int32, device="cuda")
for rep in range(2):
    call("pdas_solve_sweeps_ws", dv.ptr(cols), dv.ptr(A), dv.ptr(d), m, n, dv.ptr(ws), rep + 1,
         dv.ptr(fail), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 32)()
lib = load()
lib.pdas_debug_hop_trace.argtypes = [ctypes.c_void_p]
assert lib.pdas_debug_hop_trace(ctypes.addressof(buf)) == 0
t = [int(v) for v in buf]
z = t[0]
if not args.legacy:
    # k_casc_panel_w (warp per column): marks 0..9
    marks = [(0, "pub: columns stored (CTA barrier)"), (1, "pub: fence + flags released"),
             (2, "con: producer saw chunk-1 flag"), (3, "con: chunk-1 denominators staged"),
             (9, "con: warp 0 has the first chunk-1 stage"), (4, "con: warp 0 applied all"),
             (5, "con: triangle step 0 done"), (6, "con: chunk 0 published"),
             (7, "con: triangle step 7 done"), (8, "con: all columns stored")]
    print(f"m={m} n={n}: one warp-per-column panel hop (tile 15 -> 16, block 5), ns after "
          f"the publisher's columns are stored")
    for k, nm in marks:
        print(f"  {nm:42s} {t[k] - z:8d}")
    for w, b in ((0, 16), (7, 24)):
        print(f"  tile 16 warp {w} (clock64, both reps): work {t[b]}, stage waits {t[b + 1]}, "
              f"triangle hand-off waits {t[b + 2]}, apply steps {t[b + 3]}")
    sys.exit(0)
names = ["pub: triangle done", "pub: stored + fenced", "pub: flags released",
         "con: flag seen", "con: denominators staged", "con: chunk applied",
         "con: own triangle starts"]
print(f"m={m} n={n}: one panel hop (tile 15 -> 16, block 5), ns after the publisher's "
      f"triangle end")
for k, nm in enumerate(names):
    print(f"  {nm:28s} {t[k] - z:8d}")
tri = ["stage wait", "make_v+partials+B1", "reduce+B2", "denom+div+B3", "axpy", "publish/loop"]
tot = sum(t[8:14])
print("  tile 16's triangle, clock64 cycles summed over its 8 steps (both reps): " +
      ", ".join(f"{nm} {t[8 + i]}" for i, nm in enumerate(tri)) + f"  total {tot}")

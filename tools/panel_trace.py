"""Where the panel's time goes, from a PDAS_PANEL_TRACE=1 build (last CTA of
a 32-tile panel: waiting on predecessor tiles, applying their pivots, its own
triangle).

    make -C paper_1502_03543_b200/csrc variant VDEFS=-DPDAS_PANEL_TRACE=1 VNAME=ptrace
    PDAS_B200_LIB=paper_1502_03543_b200/csrc/build/var_ptrace/libpdas_b200.so \\
        python tools/panel_trace.py [--m 2000 --n 20000]"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

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
cols = torch.rand(m * (n + 1), dtype=torch.float64, device="cuda", generator=g) * 1e-3
d = torch.pow(10.0, torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8, device="cuda")
fail = torch.zeros(1, dtype=torch.int32, device="cuda")
call("pdas_solve_sweeps_ws", dv.ptr(cols), dv.ptr(A), dv.ptr(d), m, n, dv.ptr(ws), 1,
     dv.ptr(fail), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 8)()
lib = load()
lib.pdas_debug_panel_trace.argtypes = [ctypes.c_void_p]
assert lib.pdas_debug_panel_trace(ctypes.addressof(buf)) == 0
wait, apply, tri, na, nt = buf[0], buf[1], buf[2], buf[3], buf[4]
print(f"m={m} n={n}: last CTA of a 32-tile panel, cycles: wait {wait}  apply {apply} "
      f"({apply / max(na, 1):.0f}/step over {na})  triangle {tri} ({tri / max(nt, 1):.0f}/step "
      f"over {nt})")
steps = sum(buf[4:8]) and na  # apply-phase steps of the traced CTA (incl. its own block's)
names = ["stage wait", "make_v+partials+B1", "refill+reduce+B2", "load_p+axpy"]
tot = sum(buf[4:8])
print("  apply-step split (all apply_impl calls of that CTA):",
      ", ".join(f"{nm} {100 * buf[4 + i] / max(tot, 1):.0f}%" for i, nm in enumerate(names)))

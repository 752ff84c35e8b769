"""Per-pivot phase timeline of the warp-specialized update kernel (one CTA),
from a PDAS_WS_TRACE=1 build:

    make -C paper_1502_03543_b200/csrc variant VDEFS=-DPDAS_WS_TRACE=1 VNAME=trace
    PDAS_B200_LIB=paper_1502_03543_b200/csrc/build/var_trace/libpdas_b200.so \
        python tools/ws_trace.py [--m 2000 --n 4000]

Runs one cascade; prints, per pivot (cycles): compute C1 (axpy B + partials B),
compute wait at GA, compute C2 (axpy A + partials A), reducer wait at PA,
reducer R1 (reduce A), stage wait, reducer wait at PB, reducer R2."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200._lib import call, load  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2000)
ap.add_argument("--n", type=int, default=4000)
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
KB = 256  # kMaxBlock in cascade.cu (trace rows per role)
buf = (ctypes.c_longlong * (2 * KB * 6))()
lib = load()
lib.pdas_debug_ws_trace.argtypes = [ctypes.c_void_p]
assert lib.pdas_debug_ws_trace(ctypes.addressof(buf)) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(2, KB, 6).astype(np.float64)
C, Rd = t[0], t[1]
rows = []
for j in range(1, KB - 2):
    c1 = C[j, 2] - C[j, 1]           # after GB -> after PB arrive
    wga = C[j, 3] - C[j, 2]          # waiting for GA
    c2 = C[j, 4] - C[j, 3]           # C2 work
    wgb = C[j + 1, 1] - C[j + 1, 0]  # waiting for GB (next C1)
    wpa = Rd[j, 1] - Rd[j, 0]
    r1 = Rd[j, 2] - Rd[j, 1]
    stw = Rd[j, 3] - Rd[j, 2]
    wpb = Rd[j, 4] - Rd[j, 3]
    r2 = Rd[j, 5] - Rd[j, 4]
    per = C[j + 1, 1] - C[j, 1]
    rows.append((per, c1, wga, c2, wgb, wpa, r1, stw, wpb, r2))
a = np.array(rows)
names = ["period", "C1", "wait GA", "C2", "wait GB", "R wait PA", "R1", "stage wait",
         "R wait PB", "R2"]
print(f"m={m} n={n}: median cycles per pivot over pivots 1..{KB - 3} of one CTA's last update")
for k, nm in enumerate(names):
    print(f"  {nm:11s} median {np.median(a[:, k]):8.0f}   p90 {np.percentile(a[:, k], 90):8.0f}")

"""Time the Egidi-Maponi cascade alone (pdas_solve_sweeps_ws) with CUDA events.

    python tools/cascade_time.py [--m 2000 --n 20000 --reps 3]

Inputs are synthetic ([Y | x] random, d = 10^U[-1,1]); the cascade's cost
does not depend on the values."""
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
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
m, n = args.m, args.n
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
Y = torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g) * 1e-3
x0 = torch.rand(m, dtype=torch.float64, device="cuda", generator=g)
d = torch.pow(10.0, torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
cols = torch.empty(m * (n + 1), dtype=torch.float64, device="cuda")
ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8, device="cuda")
fail = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
E = m * n * (n + 1) // 2
for rep in range(args.reps + 1):
    cols[: m * n].copy_(Y)
    cols[m * n:].copy_(x0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    call("pdas_solve_sweeps_ws", dv.ptr(cols), dv.ptr(A), dv.ptr(d), m, n, dv.ptr(ws), rep + 1,
         dv.ptr(fail), st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if rep:
        print(f"m={m} n={n} cascade {ms:.2f} ms  {4 * E / ms / 1e9:.2f} TFLOP/s  "
              f"{16 * E / ms / 1e6:.0f} GB/s-equiv  fail={int(fail.item())}  "
              f"B={int(load().pdas_cascade_solve_block())}", flush=True)

"""CUDA-event breakdown of one PDAS iteration (default c3; --m/--n for others).

    python tools/iter_breakdown.py [--m 50 --n 200]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1502_03543_b200 as P  # noqa: E402
from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200._lib import OFF_CASCADE_FAIL, call  # noqa: E402
from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver, d_mat_vec, d_solve_many  # noqa: E402

import argparse

ap = argparse.ArgumentParser()
ap.add_argument('--m', type=int, default=2000)
ap.add_argument('--n', type=int, default=20000)
args = ap.parse_args()
m, n = args.m, args.n
lp, start = P.gen_random_feasible(m, n, 0)
prob = DeviceProblem.from_lp(lp)
eng = DeviceSolver(prob, L0=prob.validate())
st = torch.cuda.current_stream()
for rep in range(3):
    eng.load_iterate(start.x, start.y, start.s)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    h0 = time.perf_counter()
    ev[0].record(st)
    call("pdas_iter_reset", eng._sptr(), st.cuda_stream)
    call("pdas_iter_scaling", dv.ptr(eng.x), dv.ptr(eng.s), n, dv.ptr(eng.d), eng._sptr(), st.cuda_stream)
    d_mat_vec(prob.A, m, n, eng.x, eng.rhs)
    ev[1].record(st)
    eng.cols[:m * n].copy_(eng.basis.Y, non_blocking=True)
    eng.xcol.copy_(eng.rhs, non_blocking=True)
    ev[2].record(st)
    d_solve_many(eng.basis.L0, m, eng.xcol, 1)
    ev[3].record(st)
    eng.epoch += 1
    h1 = time.perf_counter()
    call("pdas_solve_sweeps_ws", dv.ptr(eng.cols), dv.ptr(prob.A), dv.ptr(eng.d), m, n,
         dv.ptr(eng.casc_ws), eng.epoch, eng._sptr(OFF_CASCADE_FAIL), st.cuda_stream)
    h2 = time.perf_counter()
    ev[4].record(st)
    eng.dy = eng.xcol
    eng._tail(eng.dy)
    ev[5].record(st)
    s_ = eng._fetch_state()
    h3 = time.perf_counter()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
    print(f"rep {rep}: scaling+rhs {ms[0]:.2f} | Y copy {ms[1]:.2f} | x0 solve {ms[2]:.2f} | "
          f"cascade {ms[3]:.2f} | tail {ms[4]:.2f} ms | host enqueue cascade {1e3*(h2-h1):.1f} ms, "
          f"wall {1e3*(h3-h0):.1f} ms, alpha {s_.alpha!r}", flush=True)

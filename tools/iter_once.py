"""Run W warm-up + K PDAS iterations of the c3 workload (for ncu / nsys-less
profiling).  python tools/iter_once.py [--m 2000 --n 20000 --warmup 1 --iters 1]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2000)
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--iters", type=int, default=1)
args = ap.parse_args()

import torch  # noqa: E402

import paper_1502_03543_b200 as P  # noqa: E402
from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver  # noqa: E402

lp, start = P.gen_random_feasible(args.m, args.n, 0)
prob = DeviceProblem.from_lp(lp)
eng = DeviceSolver(prob, L0=prob.validate())
for i in range(args.warmup + args.iters):
    eng.load_iterate(start.x, start.y, start.s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = eng.iterate()
    print(f"iter {i}: {1e3 * (time.perf_counter() - t0):.1f} ms alpha {r.state.alpha!r}", flush=True)

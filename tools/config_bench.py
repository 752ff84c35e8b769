"""Per-config timing beside the reference's compiled CPU core: one PDAS
iteration (iteration 1 from the generator's start) of each BASELINE config on
the GPU, and the reference core's cascade rate on a bounded sample of the same
iteration, extrapolated by element-steps (the cascade is > 99 % of a CPU
iteration).

    python tools/config_bench.py [--configs c1,c2,c3,c4,c5] [--cpu-seconds 5]

c5 here is gen_random_feasible(1000, 10000): the BASELINE stress instance's
D spread (1e-8..1e8) is a property of near-optimal iterates, exercised for
parity in tests/test_gpu_configs.py; per-iteration cost does not depend on D."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1502_03543_b200 as P  # noqa: E402
from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver  # noqa: E402

SHAPES = {"c1": (50, 200), "c2": (500, 5000), "c3": (2000, 20000), "c4": (1000, 100000),
          "c5": (1000, 10000)}

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
ap.add_argument("--cpu-seconds", type=float, default=5.0)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

from oracle import oracle as O  # noqa: E402  (CPU reference leg only)

core = O.reference() or O.restated()
kind = "reference core" if O.reference() else "restated oracle"
threads = os.cpu_count() or 1
print(f"{'cfg':4s} {'m':>5s} {'n':>7s} {'GPU ms/it':>10s} {'CPU ms/it':>12s} {'speed-up':>9s}   "
      f"(CPU: {kind}, {threads} threads)")
for name in args.configs.split(","):
    m, n = SHAPES[name]
    lp, start = P.gen_random_feasible(m, n, 0)
    prob = DeviceProblem.from_lp(lp)
    eng = DeviceSolver(prob, L0=prob.validate())
    x0, y0, s0 = dv.upload(start.x), dv.upload(start.y), dv.upload(start.s)
    times = []
    for i in range(args.reps + 1):
        eng.x.copy_(x0)
        eng.y.copy_(y0)
        eng.s.copy_(s0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.iterate()
        e1.record()
        torch.cuda.synchronize()
        if i:
            times.append(e0.elapsed_time(e1))
    gpu_ms = float(np.median(times))
    # CPU: cascade steps [0, k) of iteration 1, k sized to ~cpu-seconds
    a = lp.A.as_2d()
    yb = dv.download(eng.basis.Y).reshape((m, n), order="F")
    d = dv.download(eng.d)
    cols = np.empty((m, n + 1), order="F")
    E = m * n * (n + 1) // 2
    k = min(n, 64)
    while True:
        cols[:, :n] = yb
        cols[:, n] = 0.0
        dd = np.where(np.arange(n) < k, d, 1.0)
        t0 = time.perf_counter()
        core.solve_sweeps(cols, a, dd, np.zeros(n + 1), np.zeros(m), threads)
        dt = time.perf_counter() - t0
        es = sum(m * (n + 1 - l) for l in range(k))
        t_est = dt / es * E
        k2 = min(n, int(k * args.cpu_seconds / max(dt, 1e-4)))
        if k == n or k2 < 1.5 * k:
            break
        k = k2
    cpu_ms = 1e3 * t_est
    print(f"{name:4s} {m:5d} {n:7d} {gpu_ms:10.2f} {cpu_ms:12.1f} {cpu_ms / gpu_ms:8.0f}x",
          flush=True)
    del eng, prob
    torch.cuda.empty_cache()

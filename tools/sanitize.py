"""Small cascade runs for compute-sanitizer (racecheck / synccheck / memcheck):
every kernel schedule of the product path at a size the tools finish quickly.

    compute-sanitizer --tool racecheck python tools/sanitize.py
    compute-sanitizer --tool synccheck python tools/sanitize.py

Covers: the tile-width / thread layouts of m in {50, 300, 2000} (single-group
update, warp-specialized update at 128 and 256 compute threads, the panel with
its TMA ring, the fused x0 lane), a breakdown inside a later pivot block, and
the virtual-rank fused exchange of dist.py (panel peer stores + peer waits).
Each run is checked against the CPU oracle so a race that changes results
also fails here."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200._lib import call, load  # noqa: E402

K = O.restated()


def cascade(m, n, seed, x0=False, breakdown_at=None):
    rng = np.random.default_rng(seed)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    cols = np.asfortranarray(rng.uniform(-1, 1, (m, n + 1)) / np.sqrt(m))
    d = np.power(10.0, rng.uniform(-1, 1, n))
    d[rng.random(n) < 0.1] = 1.0
    if breakdown_at is not None:
        c = cols.copy(order="F")
        assert K.solve_sweeps_prefix(c, a, d, np.zeros(n + 1), np.zeros(m), breakdown_at, 1) == 0
        q = K.dot_tree(a[:, breakdown_at], c[:, breakdown_at])
        d[breakdown_at] = 1.0 - 1.0 / q
    ref = cols.copy(order="F")
    ret = K.solve_sweeps(ref, a, d, np.zeros(n + 1), np.zeros(m), 1)
    dc, da, dd = dv.upload(cols), dv.upload(a), dv.upload(d)
    ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8,
                     device=dv.device())
    fail = torch.zeros(1, dtype=torch.int32, device=dv.device())
    if x0:
        # x0 lane: column n holds the rhs; the library solves x0 = L^-T L^-1 rhs
        g = np.asfortranarray(a @ a.T)
        low = np.asfortranarray(np.linalg.cholesky(g))
        rhs = rng.uniform(-1, 1, m)
        cols[:, n] = rhs
        dc = dv.upload(cols)
        call("pdas_solve_sweeps_ws_x0", dv.ptr(dc), dv.ptr(da), dv.ptr(dd), dv.ptr(dv.upload(low)),
             m, n, dv.ptr(ws), 1, dv.ptr(fail), dv.stream())
        dv.synchronize()
        print(f"m={m} n={n} x0 lane: fail={int(fail.item())}", flush=True)
        return
    call("pdas_solve_sweeps_ws", dv.ptr(dc), dv.ptr(da), dv.ptr(dd), m, n, dv.ptr(ws), 1,
         dv.ptr(fail), dv.stream())
    dv.synchronize()
    f = int(fail.item())
    ok = f == ret and (ret != 0 or np.array_equal(
        dv.download(dc).view(np.uint64), ref.ravel(order="F").view(np.uint64)))
    print(f"m={m} n={n} fail={f} ref={ret} {'OK' if ok else 'MISMATCH'}", flush=True)
    assert ok


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for m, n in ((50, 300), (300, 600), (2000, 600)):
        cascade(m, n, 1)
    cascade(300, 1100, 2, breakdown_at=700)
    cascade(2000, 600, 3, x0=True)
    if "--no-dist" not in sys.argv:
        import pytest

        sys.exit(pytest.main(["-q", "-p", "no:cacheprovider", "-x",
                              "tests/test_gpu_dist.py::test_virtual_ranks_fused_exchange_bitwise"]))

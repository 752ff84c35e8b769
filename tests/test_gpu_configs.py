"""BASELINE configs c4 and c5 at their real sizes on the GPU, checked against
the CPU oracle (the reference's compiled core when oracle/_ref is built, else
the C restatement, all host threads).

* c5 (m=1000, n=10000, D spanning 1e-8..1e8 -- the fp64 stability stress):
  the whole cascade, every byte of [Y | x] and the return code.
* c4 (m=1000, n=100000, Y ~ 800 MB): head, middle and tail windows of 256
  pivots in one cascade over all 100001 columns (d = 1 skips the rest, exactly
  as in the reference), then the full 100000-step cascade twice for
  run-to-run bit determinism.
"""

import os

import numpy as np
import pytest

from conftest import bits_equal
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _core():
    return O.reference() or O.restated()


def _gpu_cascade(cols, a, d):
    import torch
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200._lib import call, load

    m, n = a.shape
    dc, da, dd = dv.upload(cols), dv.upload(a), dv.upload(d)
    ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8,
                     device=dv.device())
    fail = torch.zeros(1, dtype=torch.int32, device=dv.device())
    call("pdas_solve_sweeps_ws", dv.ptr(dc), dv.ptr(da), dv.ptr(dd), m, n, dv.ptr(ws), 1,
         dv.ptr(fail), dv.stream())
    dv.synchronize()
    return int(fail.item()), dc


def _basis(gpu, a):
    """Y = (AA^T)^-1 A on the device (bitwise the oracle's: test_gpu_kernels)."""
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200.engine import DeviceProblem, prepare_basis

    m, n = a.shape
    prob = DeviceProblem(a, np.zeros(m), np.zeros(n), m, n)
    basis = prepare_basis(prob)
    return dv.download(basis.Y).reshape((m, n), order="F")


def test_c5_stress_cascade_bitwise(gpu):
    m, n = 1000, 10000
    rng = np.random.default_rng(55)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = np.power(10.0, rng.uniform(-8, 8, n))
    y = _basis(gpu, a)
    cols = np.asfortranarray(np.column_stack([y, rng.uniform(-1, 1, m)]))
    ref = cols.copy(order="F")
    ret = _core().solve_sweeps(ref, a, d, np.zeros(n + 1), np.zeros(m), os.cpu_count() or 1)
    fail, dc = _gpu_cascade(cols, a, d)
    assert fail == ret
    if ret == 0:
        from paper_1502_03543_b200 import _device as dv

        assert bits_equal(dv.download(dc).reshape((m, n + 1), order="F"), ref)


def test_c4_wide_windows_and_determinism(gpu):
    """c4 beyond the prefix: three 256-pivot windows -- head [0, 256), middle
    [49920, 50176) and tail [99744, 100000) (the last pivot block, the x
    column's tile) -- active in ONE cascade over all 100001 columns, d = 1
    (exact skips, _kernels.pyx:242-243) elsewhere; every byte of [Y | x] and
    the return code against the reference core.  Then the full 100000-step
    cascade twice for run-to-run bit determinism."""
    from paper_1502_03543_b200 import _device as dv

    m, n, k = 1000, 100000, 256
    rng = np.random.default_rng(44)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    cols = np.asfortranarray(rng.uniform(-1, 1, (m, n + 1)) / np.sqrt(m))
    d = np.power(10.0, rng.uniform(-2, 2, n))
    idx = np.arange(n)
    live = (idx < k) | ((idx >= 49920) & (idx < 49920 + k)) | (idx >= n - k)
    dk = np.where(live, d, 1.0)
    ref = cols.copy(order="F")
    ret = _core().solve_sweeps(ref, a, dk, np.zeros(n + 1), np.zeros(m), os.cpu_count() or 1)
    fail, dc = _gpu_cascade(cols, a, dk)
    assert fail == ret == 0
    got = dv.download(dc)
    assert bits_equal(got, ref.ravel(order="F"))
    # the windows really moved the columns they reach
    assert not bits_equal(ref[:, n], cols[:, n]) and bits_equal(ref[:, :1], cols[:, :1])
    del got, ref
    f1, c1 = _gpu_cascade(cols, a, d)
    h1 = dv.download(c1)
    del c1
    f2, c2 = _gpu_cascade(cols, a, d)
    assert f1 == f2
    assert bits_equal(dv.download(c2), h1)


def test_c5_near_optimal_iterate_bitwise(gpu):
    """BASELINE configs[4] as SURVEY §8(d)(ii) defines it: the reference's own
    iterate of gen_random_feasible(1000, 10000, 0) at the first iteration
    where max d / min d >= 1e16 (tests/golden/c5_nearopt.npz, iteration 40),
    then two PDAS iterations on the GPU: dy, the ratio test's blocking index,
    the trace row and the new iterate, bit for bit."""
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver
    from conftest import load_golden, sha

    P = gpu
    g = load_golden("c5_nearopt.npz")
    lp, _ = P.gen_random_feasible(1000, 10000, 0)
    assert sha(lp.A.data) == str(g["A_sha"])
    assert sha(lp.b) == str(g["b_sha"]) and sha(lp.c) == str(g["c_sha"])
    d = g["x"] / g["s"]
    assert d.max() / d.min() >= 1e16
    eng = DeviceSolver(DeviceProblem.from_lp(lp))
    eng.load_iterate(g["x"], g["y"], g["s"])
    for it in range(len(g["trace"])):
        res = eng.iterate()
        st = res.state
        assert bits_equal(dv.download(eng.dy), g["dy"][it]), it
        assert int(st.blocking) == int(g["blocking"][it])
        row = [st.gap, st.alpha, st.pobj, st.dobj, st.r_primal, st.r_dual, st.r_comp,
               float(st.fallback)]
        assert bits_equal(np.array(row), g["trace"][it]), it
        x, y, s = eng.read_iterate()
        assert [sha(x), sha(y), sha(s)] == list(g["iter_sha"][it]), it

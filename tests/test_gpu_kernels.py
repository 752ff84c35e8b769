"""CUDA kernel table vs the reference: bitwise parity on the golden vectors
the unmodified reference produced (tests/golden/kernels.npz), the SPEC worked
examples, and randomized cascades checked against the CPU oracle."""

import numpy as np
import pytest

from conftest import bits_equal
from oracle import oracle as O
import spec_cases as SC

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K(gpu):
    assert gpu.active_core() == "cuda-sm_100a"
    from paper_1502_03543_b200._core import kernels

    return kernels


@pytest.mark.parametrize("case", SC.CASES, ids=[c.__name__ for c in SC.CASES])
def test_spec_examples(K, case):
    case(K)


def test_dot_tree_all_lengths(K, kernels_golden):
    g = kernels_golden
    n = 0
    for key in g.files:
        if key.startswith("dot/") and key.endswith("/r"):
            base = key[:-2]
            assert bits_equal(K.dot_tree(g[base + "/u"], g[base + "/v"]), g[key]), key
            n += 1
    assert n > 140


def test_golden_kernels(K, kernels_golden):
    g = kernels_golden
    for tag in g["_names"]:
        tag = str(tag)
        a, x, y, d = (g[f"{tag}/{k}"] for k in ("A", "x", "y", "d"))
        a = np.asfortranarray(a)
        assert bits_equal(K.mat_vec(a, x), g[f"{tag}/mat_vec"]), tag
        assert bits_equal(K.mat_t_vec(a, y), g[f"{tag}/mat_t_vec"]), tag
        assert bits_equal(K.gram(a), g[f"{tag}/gram"]), tag
        sgm = K.scaled_gram(a, d)
        assert bits_equal(sgm, g[f"{tag}/scaled_gram"]), tag
        low, fail = K.cholesky_factor(sgm, 1e-12)
        assert fail == int(g[f"{tag}/chol_fail"]), tag
        assert bits_equal(low, g[f"{tag}/chol_L"]), tag
        low0, fail0 = K.cholesky_factor(np.asfortranarray(g[f"{tag}/gram"]), 1e-12)
        assert fail0 == int(g[f"{tag}/chol0_fail"]), tag
        assert bits_equal(low0, g[f"{tag}/chol0_L"]), tag
        if f"{tag}/solve_X" in g:
            xs = K.cholesky_solve_many(low, np.asfortranarray(g[f"{tag}/solve_B"]))
            assert bits_equal(xs, g[f"{tag}/solve_X"]), tag
        if f"{tag}/casc_out" in g:
            assert bits_equal(K.cholesky_solve_many(low0, a), g[f"{tag}/Y"]), tag
            cols = np.asfortranarray(g[f"{tag}/casc_in"]).copy(order="F")
            m, n = a.shape
            ret = K.solve_sweeps(cols, a, d, np.zeros(n + 1), np.zeros(m), 1)
            assert ret == int(g[f"{tag}/casc_ret"]), tag
            assert bits_equal(cols, g[f"{tag}/casc_out"]), tag


def test_breakdown_return_codes(K, kernels_golden):
    g = kernels_golden
    for tag in ("bd1", "bd3", "bd_skip"):
        a = np.asfortranarray(g[f"{tag}/A"])
        cols = np.asfortranarray(g[f"{tag}/casc_in"]).copy(order="F")
        ret = K.solve_sweeps(cols, a, g[f"{tag}/d"], np.zeros(4), np.zeros(3), 1)
        assert ret == int(g[f"{tag}/casc_ret"]), tag


def _oracle_cascade(a, d, rhs):
    R = O.restated()
    basis = O.prepare_woodbury(R, a)
    cols, inner, v = O.init_workspace(R, basis, rhs)
    cin = cols.copy(order="F")
    ret = R.solve_sweeps(cols, a, d, inner, v, 8)
    return cin, cols, ret


# every tile configuration of cascade.cu (H = 1 .. 1024) plus odd m (no-TMA
# path), n not a multiple of the tile width or of the pivot block, skips
@pytest.mark.parametrize("m,n", [(1, 1), (1, 9), (2, 3), (3, 70), (7, 8), (31, 65), (32, 200),
                                 (33, 41), (64, 130), (65, 129), (100, 300), (129, 260),
                                 (255, 300), (257, 400), (511, 520), (513, 600), (1000, 1100),
                                 (1024, 1030), (1025, 1040), (2000, 2100)])
def test_cascade_random_vs_oracle(K, m, n):
    rng = np.random.default_rng(1000 * m + n)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = np.power(10.0, rng.uniform(-3, 3, n))
    d[rng.random(n) < 0.1] = 1.0
    rhs = rng.uniform(-1, 1, m)
    cin, cref, ret = _oracle_cascade(a, d, rhs)
    cols = cin.copy(order="F")
    got = K.solve_sweeps(cols, a, d, np.zeros(n + 1), np.zeros(m), 1)
    assert got == ret
    if ret == 0:
        assert bits_equal(cols, cref)


def test_cascade_wide_d_spread(K):
    """c5-style stress: d = 10^U[-8,8]."""
    rng = np.random.default_rng(5)
    m, n = 50, 400
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = np.power(10.0, rng.uniform(-8, 8, n))
    rhs = rng.uniform(-1, 1, m)
    cin, cref, ret = _oracle_cascade(a, d, rhs)
    cols = cin.copy(order="F")
    assert K.solve_sweeps(cols, a, d, np.zeros(n + 1), np.zeros(m), 1) == ret
    if ret == 0:
        assert bits_equal(cols, cref)


@pytest.mark.parametrize("m,n", [(1, 1), (3, 5), (40, 45), (64, 64), (100, 70), (300, 500)])
def test_mat_vec_gram_chol_random_vs_oracle(K, m, n):
    R = O.restated()
    rng = np.random.default_rng(m * 7 + n)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    x = rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, m)
    d = np.power(10.0, rng.uniform(-3, 3, n))
    assert bits_equal(K.mat_vec(a, x), R.mat_vec(a, x))
    assert bits_equal(K.mat_t_vec(a, y), R.mat_t_vec(a, y))
    g = R.scaled_gram(a, d)
    assert bits_equal(K.scaled_gram(a, d), g)
    l1, f1 = K.cholesky_factor(g, 1e-12)
    l2, f2 = R.cholesky_factor(g, 1e-12)
    assert f1 == f2 and bits_equal(l1, l2)
    if f2 < 0:
        B = np.asfortranarray(rng.uniform(-1, 1, (m, 37)))
        assert bits_equal(K.cholesky_solve_many(l2, B), R.cholesky_solve_many(l2, B))


def test_mat_vec_long_rows(K):
    """Row trees over n up to 100000 (c4's n): k-split partials + finish."""
    R = O.restated()
    rng = np.random.default_rng(3)
    for m, n in [(5, 20000), (3, 100000), (40, 4097)]:
        a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
        x = rng.uniform(-1, 1, n)
        assert bits_equal(K.mat_vec(a, x), R.mat_vec(a, x)), (m, n)
        u = rng.uniform(-1, 1, n)
        assert K.dot_tree(u, x) == R.dot_tree(u, x)


def test_single_step_api_matches_cascade(gpu):
    """rank_one_step / parallel_sweep applied n times == solve_woodbury (bitwise)."""
    P = gpu
    rng = np.random.default_rng(2)
    A = P.DenseMatrix.from_array(rng.uniform(-1, 1, (6, 11)))
    d = np.power(10.0, rng.uniform(-2, 2, 11))
    d[3] = 1.0
    rhs = rng.uniform(-1, 1, 6)
    basis = P.prepare_woodbury(A)
    ws = P.init_workspace(basis, rhs)
    for l in range(1, 12):
        P.parallel_sweep(ws, A, d, l, workers=3)
    assert bits_equal(ws.x_column, P.solve_woodbury(basis, A, d, rhs))
    assert bits_equal(ws.x_column, P.solve_woodbury_parallel(basis, A, d, rhs, 7))


def test_hoisted_division_bits(gpu):
    """div_by(a, b, div_recip(b)) (the cascade's per-column divide, common.cuh)
    is bit-identical to the IEEE a / b: random significands over the whole
    exponent range, the denominators the cascade sees (1 + inner), and the
    special values that leave the division's fast path."""
    import torch
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200._lib import call

    rng = np.random.default_rng(2024)
    n = 1 << 22
    bits = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) | (
        rng.integers(0, 2, size=n, dtype=np.uint64) << np.uint64(63))
    a = bits.view(np.float64).copy()
    b = rng.integers(0, 1 << 63, size=n, dtype=np.uint64).view(np.float64).copy()
    k = n // 4
    a[:k] = rng.standard_normal(k) * 10.0 ** rng.uniform(-12, 12, k)
    b[:k] = 1.0 + rng.standard_normal(k) * 10.0 ** rng.uniform(-16, 4, k)
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                   1.7976931348623157e308, 1.0, -1.0, 3.0, 1e-300, 1e300, 0.5, 2.0 ** -1022,
                   2.0 ** -1074, 2.0 ** 1023, 1.0 - 2.0 ** -53, 1.0 + 2.0 ** -52])
    ga, gb = np.meshgrid(sp, sp)
    a = np.concatenate([a, ga.ravel(), sp * 3.7, sp])
    b = np.concatenate([b, gb.ravel(), sp, sp * 1e-310])
    da, db = dv.upload(a), dv.upload(b)
    fast, ref = dv.empty(a.size), dv.empty(a.size)
    call("pdas_selftest_div", dv.ptr(da), dv.ptr(db), a.size, dv.ptr(fast), dv.ptr(ref),
         dv.stream())
    f, r = dv.download(fast), dv.download(ref)
    assert f.view(np.uint64).tobytes() == r.view(np.uint64).tobytes()
    with np.errstate(all="ignore"):
        host = a / b
    ok = ~np.isnan(host)
    assert bits_equal(r[ok], host[ok])  # and both are the IEEE quotient
    del torch


@pytest.mark.parametrize("m,n", [(1, 4), (2, 9), (7, 30), (33, 70), (64, 100), (50, 200),
                                 (50, 203), (300, 1024), (300, 1030), (1000, 2048), (1000, 2050)])
def test_cascade_with_fused_x0(gpu, m, n):
    """pdas_solve_sweeps_ws_x0: x0 = L0^-T L0^-1 rhs solved inside the cascade
    call (overlapped on its own stream when column n is alone in the last tile,
    sequential otherwise) == init_workspace + solve_sweeps (normal.py:115-124)."""
    import torch
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200._lib import call, load

    rng = np.random.default_rng(m * 31 + n)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = np.power(10.0, rng.uniform(-3, 3, n))
    d[rng.random(n) < 0.1] = 1.0
    rhs = rng.uniform(-1, 1, m)
    R = O.restated()
    basis = O.prepare_woodbury(R, a)
    cref, inner, v = O.init_workspace(R, basis, rhs)
    ret = R.solve_sweeps(cref, a, d, inner, v, 8)
    cin = np.asfortranarray(np.column_stack([np.asarray(basis.Y), rhs]))
    cols = dv.upload(cin)
    ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8,
                     device=dv.device())
    fail = torch.zeros(1, dtype=torch.int32, device=dv.device())
    da, dd, dl = dv.upload(a), dv.upload(d), dv.upload(np.asfortranarray(basis.L0))  # kept alive
    call("pdas_solve_sweeps_ws_x0", dv.ptr(cols), dv.ptr(da), dv.ptr(dd), dv.ptr(dl), m, n,
         dv.ptr(ws), 1, dv.ptr(fail), dv.stream())
    dv.synchronize()
    assert int(fail.item()) == ret
    if ret == 0:
        assert bits_equal(dv.download(cols).reshape((m, n + 1), order="F"), cref)


@pytest.mark.parametrize("m", [3000, 3500, 4096, 5000])
def test_cascade_large_m_vs_oracle(gpu, m):
    """m > 2048: the 2- and 4-stage TMA rings (the 5-stage one no longer fits
    shared memory) and the R >= 8 tiles; random [Y | x] (no basis needed)."""
    n = 300
    rng = np.random.default_rng(m)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = np.power(10.0, rng.uniform(-2, 2, n))
    d[rng.random(n) < 0.1] = 1.0
    cols = np.asfortranarray(rng.uniform(-1, 1, (m, n + 1)) / np.sqrt(m))
    ref = cols.copy(order="F")
    ret = O.restated().solve_sweeps(ref, a, d, np.zeros(n + 1), np.zeros(m), 8)
    got = cols.copy(order="F")
    assert K_solve(gpu, got, a, d) == ret
    if ret == 0:
        assert bits_equal(got, ref)


def K_solve(gpu, cols, a, d):
    from paper_1502_03543_b200._core import kernels

    m, n = a.shape
    return kernels.solve_sweeps(cols, a, d, np.zeros(n + 1), np.zeros(m), 1)


@pytest.mark.parametrize("m,k", [(300, 100), (2000, 37), (2000, 1), (6500, 3), (9000, 2)])
def test_solve_many_shared_memory_backward(K, m, k):
    """cholesky_solve_many (_kernels.pyx:174-193): the forward sweep and the
    shared-memory-resident backward sweep vs the oracle, including m past the
    old 6400 limit (one resident right-hand side per CTA) and k = 1."""
    R = O.restated()
    rng = np.random.default_rng(m + k)
    low = np.tril(rng.uniform(-1, 1, (m, m))) / np.sqrt(m)
    low[np.diag_indices(m)] = rng.uniform(1.0, 2.0, m)
    low = np.asfortranarray(low)
    B = np.asfortranarray(rng.uniform(-1, 1, (m, k)))
    assert bits_equal(K.cholesky_solve_many(low, B), R.cholesky_solve_many(low, B))

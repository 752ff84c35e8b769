"""Pin the CPU oracle (oracle/) to the reference: SPEC worked examples, the
golden vectors produced by the unmodified reference (tests/golden/), and --
where oracle/_ref was built -- the reference's own compiled core."""

import os

import numpy as np
import pytest

from conftest import bits_equal, load_golden, sha
from oracle import oracle as O
import spec_cases as SC

RESTATED = O.restated()
REFERENCE = O.reference()
TABLES = [("restated", RESTATED)] + ([("reference", REFERENCE)] if REFERENCE else [])


@pytest.mark.parametrize("name,K", TABLES, ids=[t[0] for t in TABLES])
@pytest.mark.parametrize("case", SC.CASES, ids=[c.__name__ for c in SC.CASES])
def test_spec_examples(name, K, case):
    case(K)


@pytest.mark.parametrize("gap_tol,iters,obj", SC.WORKED_RUNS)
def test_worked_lp(gap_tol, iters, obj):
    w = SC.WORKED
    x, y, s, st, tr = O.solve_lp(RESTATED, w["A"], w["b"], w["c"], w["x"], w["y"], w["s"],
                                 gap_tol=gap_tol)
    assert st is O.Status.OPTIMAL
    assert len(tr) == iters
    assert abs(tr[0].alpha - SC.WORKED_ALPHA1) < 1e-15
    assert RESTATED.dot_tree(w["c"], x) == obj


def test_restated_matches_golden_kernels(kernels_golden):
    g = kernels_golden
    K = RESTATED
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
        assert fail0 == int(g[f"{tag}/chol0_fail"]) and bits_equal(low0, g[f"{tag}/chol0_L"]), tag
        if f"{tag}/solve_X" in g:
            xs = K.cholesky_solve_many(low, np.asfortranarray(g[f"{tag}/solve_B"]))
            assert bits_equal(xs, g[f"{tag}/solve_X"]), tag
        if f"{tag}/casc_out" in g:
            y_ = K.cholesky_solve_many(low0, a)
            assert bits_equal(y_, g[f"{tag}/Y"]), tag
            cols = np.asfortranarray(g[f"{tag}/casc_in"]).copy(order="F")
            m, n = a.shape
            ret = K.solve_sweeps(cols, a, d, np.zeros(n + 1), np.zeros(m), 3)
            assert ret == int(g[f"{tag}/casc_ret"]), tag
            assert bits_equal(cols, g[f"{tag}/casc_out"]), tag


def test_restated_dot_and_breakdowns(kernels_golden):
    g = kernels_golden
    for key in g.files:
        if key.startswith("dot/") and key.endswith("/r"):
            base = key[:-2]
            assert bits_equal(RESTATED.dot_tree(g[base + "/u"], g[base + "/v"]), g[key]), key
    for tag in ("bd1", "bd3", "bd_skip"):
        a = np.asfortranarray(g[f"{tag}/A"])
        cols = np.asfortranarray(g[f"{tag}/casc_in"]).copy(order="F")
        ret = RESTATED.solve_sweeps(cols, a, g[f"{tag}/d"], np.zeros(4), np.zeros(3), 1)
        assert ret == int(g[f"{tag}/casc_ret"]), tag
    assert int(g["bd1/casc_ret"]) == 1 and int(g["bd3/casc_ret"]) == 3


@pytest.mark.parametrize("seed", range(5))
def test_c1_trajectory_matches_reference(seed):
    g = load_golden(f"c1_seed{seed}.npz")
    a, b, c, x, y, s = O.gen_random_feasible(RESTATED, 50, 200, seed)
    assert sha(a.ravel(order="F")) == str(g["A_sha"])
    assert bits_equal(b, g["b"]) and bits_equal(c, g["c"])
    blocking = []
    xf, yf, sf, st, tr = O.solve_lp(RESTATED, a, b, c, x, y, s)
    assert st.value == str(g["status"])
    assert len(tr) == len(g["trace"])
    for r, gr in zip(tr, g["trace"]):
        got = [r.gap, r.alpha, r.primal_obj, r.dual_obj, r.r_primal, r.r_dual, r.r_comp,
               float(r.fallback)]
        assert bits_equal(np.array(got), gr)
        blocking.append(r.blocking)
    assert blocking == list(g["blocking"])
    assert bits_equal(xf, g["x"]) and bits_equal(yf, g["y"]) and bits_equal(sf, g["s"])


def test_c1_basis_matches_reference():
    g = load_golden("c1_seed0.npz")
    a, *_ = O.gen_random_feasible(RESTATED, 50, 200, 0)
    basis = O.prepare_woodbury(RESTATED, a)
    assert bits_equal(basis.L0, g["L0"]) and bits_equal(basis.Y, g["Y"])


def test_c2_first_iterations_match_reference():
    g = load_golden("c2_seed0.npz")
    k = O.reference() or RESTATED
    a, b, c, x, y, s = O.gen_random_feasible(k, 500, 5000, 0)
    assert sha(a.ravel(order="F")) == str(g["A_sha"])
    seen = []

    def hook(it, x_, y_, s_, dirs):
        seen.append([sha(x_), sha(y_), sha(s_)])
        if it == 1:
            assert bits_equal(dirs.dy, g["it1_dy"])

    O.solve_lp(k, a, b, c, x, y, s, max_iter=2, workers=os.cpu_count() or 1, on_iter=hook)
    assert seen == [list(r) for r in g["iter_sha"][:2]]


def test_restated_worker_count_is_bitwise_invariant():
    rng = np.random.default_rng(7)
    a, d, rhs = O.random_system(RESTATED, rng, 37, 90)
    basis = O.prepare_woodbury(RESTATED, a)
    outs = []
    for w in (1, 2, 3, 7):
        cols, inner, v = O.init_workspace(RESTATED, basis, rhs)
        assert RESTATED.solve_sweeps(cols, a, d, inner, v, w) == 0
        outs.append(cols)
    assert all(bits_equal(o, outs[0]) for o in outs)


@pytest.mark.skipif(REFERENCE is None, reason="oracle/_ref not built")
def test_restated_equals_reference_core_random():
    rng = np.random.default_rng(11)
    for m, n in [(1, 3), (2, 5), (13, 29), (64, 130)]:
        a, d, rhs = O.random_system(RESTATED, rng, m, n)
        d[rng.random(n) < 0.3] = 1.0
        b1 = O.prepare_woodbury(RESTATED, a)
        b2 = O.prepare_woodbury(REFERENCE, a)
        assert bits_equal(b1.Y, b2.Y) and bits_equal(b1.L0, b2.L0)
        c1, i1, v1 = O.init_workspace(RESTATED, b1, rhs)
        c2 = c1.copy(order="F")
        r1 = RESTATED.solve_sweeps(c1, a, d, i1, v1, 2)
        r2 = REFERENCE.solve_sweeps(c2, a, d, np.zeros(n + 1), np.zeros(m), 1)
        assert r1 == r2 and bits_equal(c1, c2)


@pytest.mark.parametrize("tag", ["bd_small", "nb_small"])
def test_oracle_rare_exits_match_reference(tag):
    """The oracle's solve_lp on the breakdown instances (tests/golden/lp_cases.py)
    reproduces the reference's fallback trajectory / NUMERICAL_BREAKDOWN exit
    (tests/golden/breakdown.npz) bit for bit."""
    import sys

    from conftest import GOLDEN

    sys.path.insert(0, GOLDEN)
    import lp_cases as LC

    g = load_golden("breakdown.npz")
    m, n, l, seed, dl, dscale = LC.CASES[tag]
    A, x, y, s = LC.breakdown_raw(m, n, l, seed, dl, dscale)
    a = np.asfortranarray(A)
    assert sha(a.ravel(order="F")) == str(g[f"{tag}/A_sha"])
    K = RESTATED
    b = K.mat_vec(a, x)
    c = K.mat_t_vec(a, y) + s
    assert bits_equal(b, g[f"{tag}/b"]) and bits_equal(c, g[f"{tag}/c"])
    xo, yo, so, st, tr = O.solve_lp(K, a, b, c, x, y, s)
    assert st.value == str(g[f"{tag}/status"])
    rows = np.array([[r.gap, r.alpha, r.primal_obj, r.dual_obj, r.r_primal, r.r_dual, r.r_comp,
                      float(r.fallback)] for r in tr]).reshape(len(tr), 8)
    assert bits_equal(rows, g[f"{tag}/trace"])
    assert [r.blocking for r in tr] == [int(v) for v in g[f"{tag}/blocking"]]
    assert bits_equal(xo, g[f"{tag}/x"]) and bits_equal(so, g[f"{tag}/s"])

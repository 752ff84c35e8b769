"""The rare exits of solve_lp on the GPU, bit for bit against the reference
(golden fixtures from tests/golden/make_golden.py breakdown, built with the
UNMODIFIED reference; instances from tests/golden/lp_cases.py).

* SingularUpdate -> solve_direct fallback (solver.py:161-165, normal.py:172-173):
  the cascade breaks down (return l+1, _kernels.pyx:254-256), the direct
  Cholesky path takes over, the trace row is flagged fallback=True, and the
  trajectory continues.  bd_small (m=20, n=60: breakdowns at steps 8 and 58)
  and bd_large (m=300, n=3000: step 701 sits in pivot block 2, so the panel
  finds it while the previous block's update kernel is still running).
* NUMERICAL_BREAKDOWN (solver.py:226-228): the fallback's Cholesky fails too.
* UNBOUNDED (solver.py:237-256): no interior point with finite directions can
  reach it -- for every j either t_j > 0 (ds_j = -t_j < 0 blocks) or
  t_j <= 0 (dx_j = d_j t_j - x_j < 0 blocks).  The branch is covered at the
  level where it is decided: the device ratio test returns CAP_ALPHA when no
  component blocks, and solve_lp maps an alpha >= CAP_ALPHA state to
  Status.UNBOUNDED with the reference's trace row.
"""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal, load_golden, sha

sys.path.insert(0, GOLDEN)
import lp_cases as LC  # noqa: E402

pytestmark = pytest.mark.gpu


def _lp(P, tag, g):
    m, n, l, seed, dl, dscale = LC.CASES[tag]
    A, x, y, s = LC.breakdown_raw(m, n, l, seed, dl, dscale)
    Af = P.DenseMatrix.from_array(np.asfortranarray(A))
    assert sha(Af.data) == str(g[f"{tag}/A_sha"])
    # the GPU's own b = A x and c = A^T y + s are the reference's bits
    b = np.asarray(P.mat_vec(Af, x))
    c = np.asarray(P.mat_t_vec(Af, y)) + s
    assert bits_equal(b, g[f"{tag}/b"]) and bits_equal(c, g[f"{tag}/c"])
    return P.StandardFormLP(Af, b, c), P.InteriorPoint(x, y, s)


def _rows(tr):
    return np.array([[r.gap, r.alpha, r.primal_obj, r.dual_obj, r.r_primal, r.r_dual, r.r_comp,
                      float(r.fallback)] for r in tr]).reshape(len(tr), 8)


@pytest.mark.parametrize("tag", ["bd_small", "bd_large"])
def test_fallback_trajectory_bitwise(gpu, tag):
    P = gpu
    g = load_golden("breakdown.npz")
    lp, start = _lp(P, tag, g)
    p, st, tr = P.solve_lp(lp, start)
    assert st.value == str(g[f"{tag}/status"])
    want = g[f"{tag}/trace"]
    assert len(tr) == len(want)
    assert want[:, 7].any() and not want[:, 7].all()  # both paths are exercised
    assert bits_equal(_rows(tr), want)
    assert bits_equal(p.x, g[f"{tag}/x"]) and bits_equal(p.y, g[f"{tag}/y"])
    assert bits_equal(p.s, g[f"{tag}/s"])


@pytest.mark.parametrize("tag", ["bd_small", "bd_large"])
def test_fallback_iterations_through_engine(gpu, tag):
    """Per iteration: the cascade's own return code (before the fallback), the
    blocking index and the iterate hashes."""
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200._lib import OFF_CASCADE_FAIL, call
    from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver

    P = gpu
    g = load_golden("breakdown.npz")
    lp, start = _lp(P, tag, g)
    eng = DeviceSolver(DeviceProblem.from_lp(lp))
    eng.load_iterate(start.x, start.y, start.s)
    rets = g[f"{tag}/cascade_ret"]
    for it in range(min(len(rets), 14)):
        # the cascade alone on this iterate: return code = the reference's
        eng.enqueue_solve()
        st = eng._fetch_state()
        assert int(st.cascade_fail) == int(rets[it]), it
        res = eng.iterate()
        assert bool(res.state.fallback) == bool(rets[it])
        assert int(res.state.blocking) == int(g[f"{tag}/blocking"][it])
        x, y, s = eng.read_iterate()
        assert [sha(x), sha(y), sha(s)] == list(g[f"{tag}/iter_sha"][it]), it


def test_numerical_breakdown_exit(gpu):
    P = gpu
    g = load_golden("breakdown.npz")
    lp, start = _lp(P, "nb_small", g)
    p, st, tr = P.solve_lp(lp, start)
    assert st.value == str(g["nb_small/status"]) == "numerical_breakdown"
    assert len(tr) == len(g["nb_small/trace"]) == 0
    # the iterate is returned untouched, as in the reference
    assert bits_equal(p.x, g["nb_small/x"]) and bits_equal(p.s, g["nb_small/s"])


def test_step_length_cap_and_reference_semantics(gpu):
    """solver.py:175-189: CAP_ALPHA when nothing blocks; otherwise rho times
    the smallest ratio over both vectors (the device ratio test)."""
    P = gpu
    rng = np.random.default_rng(3)
    n = 1000
    x, s = rng.uniform(0.5, 2, n), rng.uniform(0.5, 2, n)
    p = P.InteriorPoint(x, np.zeros(3), s)
    pos = P.Directions(rng.uniform(0, 1, n), np.zeros(3), rng.uniform(0, 1, n), 0, 0, 0)
    assert P.step_length(p, pos, 0.9) == P.solver.CAP_ALPHA
    pos.dx[5] = -0.0  # -0.0 is not < 0: still nothing blocks
    assert P.step_length(p, pos, 0.9) == P.solver.CAP_ALPHA
    for _ in range(5):
        dx, ds = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        dirs = P.Directions(dx, np.zeros(3), ds, 0, 0, 0)
        neg = dx < 0
        r = [float(np.min(-x[neg] / dx[neg]))]
        neg = ds < 0
        r.append(float(np.min(-s[neg] / ds[neg])))
        assert P.step_length(p, dirs, 0.9) == 0.9 * min(r)
    only_s = P.Directions(np.ones(n), np.zeros(3), -np.ones(n), 0, 0, 0)
    assert P.step_length(p, only_s, 0.5) == 0.5 * float(np.min(s))


def test_unbounded_exit_mapping(gpu, monkeypatch):
    """An iteration whose ratio test finds no blocking component (alpha =
    CAP_ALPHA) ends the solve as UNBOUNDED with that iteration's row appended
    and the iterate unchanged (solver.py:237-256)."""
    from paper_1502_03543_b200 import engine as E

    P = gpu
    lp, start = P.gen_random_feasible(10, 30, 2)
    real = E.DeviceSolver.iterate
    calls = {"n": 0}

    def capped(self):
        res = real(self)
        calls["n"] += 1
        if calls["n"] == 2:
            # what the device reports when no component blocks: alpha = CAP,
            # no step (k_dir_finish: stepped = 0), so x, s and gap are unchanged
            res.state.alpha = P.solver.CAP_ALPHA
        return res

    p1, st1, tr1 = P.solve_lp(lp, start, P.SolveOptions(max_iter=1))
    monkeypatch.setattr(E.DeviceSolver, "iterate", capped)
    p, st, tr = P.solve_lp(lp, start)
    assert st is P.Status.UNBOUNDED and len(tr) == 2
    assert tr[1].alpha == P.solver.CAP_ALPHA and tr[1].gap == tr[0].gap
    assert bits_equal(_rows(tr[:1]), _rows(tr1))

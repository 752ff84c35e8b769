"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (/root/reference, compiled core from oracle/_ref) in this container.

    python tests/golden/make_golden.py kernels c1 c2      # ~2 min
    python tests/golden/make_golden.py c3                  # ~5 min, 8 threads

The fixtures are the parity anchors of the oracle (tests/test_oracle.py) and
of the CUDA path (tests/test_gpu_*.py).  Arrays are stored in full where they
are small; big ones (A, x, s at c2/c3) are pinned by sha256 of their bytes,
which is exact for a bitwise contract.
"""

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from _refimport import import_reference  # noqa: E402

ad = import_reference()
K = sys.modules["adascale._kernels"]
WORKERS = int(os.environ.get("GOLDEN_WORKERS", os.cpu_count() or 1))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def f2d(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------------------
def gen_kernels():
    rng = np.random.default_rng(20260418)
    out = {}
    shapes = [(1, 1), (1, 4), (2, 3), (3, 3), (5, 9), (17, 40), (31, 33), (32, 64),
              (33, 70), (50, 200), (65, 130)]
    names = []
    for (m, n) in shapes:
        tag = f"m{m}n{n}"
        names.append(tag)
        a = f2d(rng.uniform(-1, 1, (m, n)))
        x = rng.uniform(-1, 1, n)
        y = rng.uniform(-1, 1, m)
        d = np.power(10.0, rng.uniform(-3, 3, n))
        d[rng.random(n) < 0.2] = 1.0  # exact skips (_kernels.pyx:242-243)
        out[tag + "/A"] = a
        out[tag + "/x"] = x
        out[tag + "/y"] = y
        out[tag + "/d"] = d
        out[tag + "/mat_vec"] = np.asarray(K.mat_vec(a, x))
        out[tag + "/mat_t_vec"] = np.asarray(K.mat_t_vec(a, y))
        g = np.asarray(K.gram(a))
        out[tag + "/gram"] = g
        sg = np.asarray(K.scaled_gram(a, d))
        out[tag + "/scaled_gram"] = sg
        low, fail = K.cholesky_factor(f2d(sg), 1e-12)
        out[tag + "/chol_L"] = np.asarray(low)
        out[tag + "/chol_fail"] = np.array(fail)
        low0, fail0 = K.cholesky_factor(f2d(g), 1e-12)
        out[tag + "/chol0_L"] = np.asarray(low0)
        out[tag + "/chol0_fail"] = np.array(fail0)
        if fail < 0:
            bb = f2d(rng.uniform(-1, 1, (m, 3)))
            out[tag + "/solve_B"] = bb
            out[tag + "/solve_X"] = np.asarray(K.cholesky_solve_many(f2d(low), bb))
        if fail0 < 0:
            # full cascade on the true basis [Y | x0] (normal.py:108-124)
            basis = ad.prepare_woodbury(ad.DenseMatrix.from_array(a))
            rhs = rng.uniform(-1, 1, m)
            ws = ad.init_workspace(basis, rhs)
            out[tag + "/casc_rhs"] = rhs
            out[tag + "/casc_in"] = ws.cols.copy(order="F")
            ret = K.solve_sweeps(ws.cols, a, d, ws.inner, ws.v_scratch, 1)
            out[tag + "/casc_out"] = ws.cols.copy(order="F")
            out[tag + "/casc_ret"] = np.array(ret)
            out[tag + "/Y"] = np.asarray(basis.Y.as_2d())
    # tree dots over every length 1..140 (pads, odd sizes, powers of two)
    for ln in list(range(1, 141)) + [255, 256, 257, 1000, 2000]:
        u = rng.uniform(-1, 1, ln)
        v = rng.uniform(-1, 1, ln)
        out[f"dot/{ln}/u"] = u
        out[f"dot/{ln}/v"] = v
        out[f"dot/{ln}/r"] = np.array(K.dot_tree(u, v))
    # signed-zero padding case: -0.0 products must become +0.0 at level 0
    u = np.array([-0.0, 1.0, -0.0])
    v = np.array([1.0, 0.0, 1.0])
    out["dot/signed_zero/u"], out["dot/signed_zero/v"] = u, v
    out["dot/signed_zero/r"] = np.array(K.dot_tree(u, v))
    # breakdowns: square A makes a_l^T M^{-1} a_l == 1, so d_l -> 0 breaks step l
    for tag, dvec in (("bd1", [1e-14, 2.0, 3.0]), ("bd3", [2.0, 3.0, 1e-14]),
                      ("bd_skip", [1.0, 1.0, 1e-14])):
        a = f2d(rng.uniform(-1, 1, (3, 3)))
        basis = ad.prepare_woodbury(ad.DenseMatrix.from_array(a))
        rhs = rng.uniform(-1, 1, 3)
        ws = ad.init_workspace(basis, rhs)
        out[f"{tag}/A"] = a
        out[f"{tag}/d"] = np.array(dvec)
        out[f"{tag}/casc_in"] = ws.cols.copy(order="F")
        out[f"{tag}/casc_ret"] = np.array(
            K.solve_sweeps(ws.cols, a, np.array(dvec), ws.inner, ws.v_scratch, 1))
    out["_names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("kernels.npz", len(out), "arrays")


# ---------------------------------------------------------------------------
def trajectory(m, n, seed, max_iter=500, full=True, workers=1):
    """Run the reference's own public functions (the loop of solver.py:197-279)
    recording per-iteration intermediates, then cross-check against solve_lp."""
    t0 = time.perf_counter()
    lp, start = ad.gen_random_feasible(m, n, seed)
    t_gen = time.perf_counter() - t0
    rec = {"A_sha": sha(lp.A.data), "b": lp.b, "c": lp.c, "x0": start.x, "y0": start.y,
           "s0": start.s, "t_gen": np.array(t_gen)}
    t0 = time.perf_counter()
    backend = ad.solver.make_backend(lp, "woodbury", workers)
    rec["t_prepare"] = np.array(time.perf_counter() - t0)
    if full:
        rec["L0"] = np.asarray(backend.basis.L0.as_2d())
        rec["Y"] = np.asarray(backend.basis.Y.as_2d())
    else:
        rec["L0_sha"] = sha(backend.basis.L0.data)
        rec["Y_sha"] = sha(backend.basis.Y.data)
    p = start.copy()
    gap = ad.duality_gap(p)
    gap_tol = ad.solver.GAP_TOL_REL * (1.0 + abs(ad.dot_tree(lp.c, p.x)))
    rows, blocking, shas, t_iter = [], [], [], []
    status = "iter_limit"
    for it in range(1, max_iter + 1):
        t1 = time.perf_counter()
        d = ad.scaling_diag(p)
        rhs = ad.mat_vec(lp.A, p.x)
        dirs = ad.compute_directions(lp, p, backend)
        alpha = ad.step_length(p, dirs, 0.9)
        # blocking index: first argmin over [x ratios | s ratios]
        r = np.full(2 * n, np.inf)
        neg = dirs.dx < 0
        r[:n][neg] = -p.x[neg] / dirs.dx[neg]
        neg = dirs.ds < 0
        r[n:][neg] = -p.s[neg] / dirs.ds[neg]
        blocking.append(int(np.argmin(r)) if np.isfinite(r).any() else -1)
        if it == 1:
            rec["it1_d"], rec["it1_rhs"] = d, rhs
            rec["it1_dy"], rec["it1_dx"], rec["it1_ds"] = dirs.dy, dirs.dx, dirs.ds
            if full:
                rec["it1_x0col"] = ad.linalg.cholesky_solve(backend.basis.L0, rhs)
        if alpha >= ad.solver.CAP_ALPHA:
            status = "unbounded"
            break
        p.x += alpha * dirs.dx
        p.y += alpha * dirs.dy
        p.s += alpha * dirs.ds
        gap = ad.duality_gap(p)
        t_iter.append(time.perf_counter() - t1)
        rows.append([gap, alpha, ad.dot_tree(lp.c, p.x), ad.dot_tree(lp.b, p.y),
                     dirs.residual_primal, dirs.residual_dual, dirs.residual_comp,
                     float(dirs.fallback)])
        shas.append([sha(p.x), sha(p.y), sha(p.s)])
        print(f"  it {it} gap {gap:.3e} alpha {alpha:.6f} ({t_iter[-1]:.2f}s)", flush=True)
        if gap <= gap_tol:
            status = "optimal"
            break
    rec["trace"] = np.array(rows)  # gap, alpha, pobj, dobj, r_p, r_d, r_c, fallback
    rec["blocking"] = np.array(blocking)
    rec["iter_sha"] = np.array(shas)
    rec["t_iter"] = np.array(t_iter)
    rec["status"] = np.array(status)
    rec["gap_tol"] = np.array(gap_tol)
    rec["x"], rec["y"], rec["s"] = p.x, p.y, p.s
    if max_iter >= 500:
        # cross-check: the reference's solve_lp lands on the same bits
        q, st, tr = ad.solve_lp(lp, start, ad.SolveOptions(workers=workers))
        assert st.value == status and len(tr) == len(rows), (st, len(tr))
        assert np.array_equal(q.x, p.x) and np.array_equal(q.y, p.y) and np.array_equal(q.s, p.s)
        assert [t.gap for t in tr] == [r_[0] for r_ in rows]
    return rec


def gen_c1():
    for seed in range(5):
        rec = trajectory(50, 200, seed, full=True)
        np.savez_compressed(os.path.join(HERE, f"c1_seed{seed}.npz"), **rec)
        print("c1 seed", seed, rec["status"], len(rec["trace"]), repr(rec["trace"][-1][2]))


def gen_c2():
    rec = trajectory(500, 5000, 0, full=False, workers=WORKERS)
    for k in ("x", "s", "it1_dx", "it1_ds", "it1_d", "x0", "s0", "c"):
        rec.pop(k)  # n-length arrays: pinned by sha below instead
    np.savez_compressed(os.path.join(HERE, "c2_seed0.npz"), **rec)
    print("c2", rec["status"], len(rec["trace"]))


def gen_c3():
    rec = trajectory(2000, 20000, 0, max_iter=1, full=False, workers=WORKERS)
    rec["it1_dx_sha"] = np.array(sha(rec.pop("it1_dx")))
    rec["it1_ds_sha"] = np.array(sha(rec.pop("it1_ds")))
    rec["it1_d_sha"] = np.array(sha(rec.pop("it1_d")))
    for k in ("x", "s", "x0", "s0", "c"):
        rec[k + "_sha"] = np.array(sha(rec.pop(k)))
    rec["workers"] = np.array(WORKERS)
    np.savez_compressed(os.path.join(HERE, "c3_seed0_it1.npz"), **rec)
    print("c3 it1 done", rec["t_prepare"], rec["t_iter"])


def _blocking(p, dirs, n):
    r = np.full(2 * n, np.inf)
    neg = dirs.dx < 0
    r[:n][neg] = -p.x[neg] / dirs.dx[neg]
    neg = dirs.ds < 0
    r[n:][neg] = -p.s[neg] / dirs.ds[neg]
    return int(np.argmin(r)) if np.isfinite(r).any() else -1


def gen_c5(spread=1e16, follow=2):
    """BASELINE configs[4] / SURVEY §8(d)(ii): the ill-conditioned NEAR-OPTIMAL
    iterate.  Runs the reference's own iteration (solver.py:222-278) on
    gen_random_feasible(1000, 10000, 0) until max d / min d >= `spread`,
    stores that iterate (the c5 stress point) and the next `follow`
    iterations (dy, trace row, blocking index, iterate hashes)."""
    m, n = 1000, 10000
    lp, start = ad.gen_random_feasible(m, n, 0)
    backend = ad.solver.make_backend(lp, "woodbury", WORKERS)
    p = start.copy()
    gap_tol = ad.solver.GAP_TOL_REL * (1.0 + abs(ad.dot_tree(lp.c, p.x)))
    rec = {"A_sha": sha(lp.A.data), "b_sha": sha(lp.b), "c_sha": sha(lp.c),
           "gap_tol": np.array(gap_tol), "workers": np.array(WORKERS)}
    it, hit = 0, None
    while True:
        it += 1
        d = ad.scaling_diag(p)
        sp = float(d.max() / d.min())
        if hit is None and sp >= spread:
            hit = it
            rec["start_it"] = np.array(it)  # the stored iterate is the input of iteration `it`
            rec["start_spread"] = np.array(sp)
            rec["x"], rec["y"], rec["s"] = p.x.copy(), p.y.copy(), p.s.copy()
            rows, dys, blocking, shas = [], [], [], []
        t1 = time.perf_counter()
        dirs = ad.compute_directions(lp, p, backend)
        alpha = ad.step_length(p, dirs, 0.9)
        if hit is not None:
            blocking.append(_blocking(p, dirs, n))
            dys.append(dirs.dy.copy())
        assert alpha < ad.solver.CAP_ALPHA
        p.x += alpha * dirs.dx
        p.y += alpha * dirs.dy
        p.s += alpha * dirs.ds
        gap = ad.duality_gap(p)
        print(f"  c5 it {it} spread {sp:.3e} gap {gap:.3e} alpha {alpha:.6f} fallback "
              f"{dirs.fallback} ({time.perf_counter() - t1:.1f}s)", flush=True)
        if hit is not None:
            rows.append([gap, alpha, ad.dot_tree(lp.c, p.x), ad.dot_tree(lp.b, p.y),
                         dirs.residual_primal, dirs.residual_dual, dirs.residual_comp,
                         float(dirs.fallback)])
            shas.append([sha(p.x), sha(p.y), sha(p.s)])
            if len(rows) == follow:
                break
        assert gap > gap_tol, "converged before reaching the spread"
    rec["trace"] = np.array(rows)
    rec["dy"] = np.array(dys)
    rec["blocking"] = np.array(blocking)
    rec["iter_sha"] = np.array(shas)
    np.savez_compressed(os.path.join(HERE, "c5_nearopt.npz"), **rec)
    print("c5 near-optimal: iterate", hit, "spread", rec["start_spread"])


def gen_breakdown():
    """The rare exits of solve_lp (solver.py:161-165, 226-235) on the seeded
    instances of lp_cases.py, run through the reference's own solve_lp plus
    the per-iteration loop (for the blocking index and iterate hashes)."""
    import lp_cases as LC

    out = {}
    for tag, (m, n, l, seed, dl, dscale) in LC.CASES.items():
        A, x, y, s = LC.breakdown_raw(m, n, l, seed, dl, dscale)
        Af = ad.DenseMatrix.from_array(np.asfortranarray(A))
        b = np.asarray(ad.mat_vec(Af, x))
        c = np.asarray(ad.mat_t_vec(Af, y)) + s
        lp = ad.StandardFormLP(Af, b, c)
        start = ad.InteriorPoint(x.copy(), y.copy(), s.copy())
        q, st, tr = ad.solve_lp(lp, start, ad.SolveOptions(workers=WORKERS))
        # the same loop by hand: blocking index and iterate hashes per iteration
        backend = ad.solver.make_backend(lp, "woodbury", WORKERS)
        p = start.copy()
        blocking, shas, cascade_ret = [], [], []
        for it in range(len(tr)):
            d = ad.scaling_diag(p)
            rhs = ad.mat_vec(lp.A, p.x)
            ws = ad.init_workspace(backend.basis, rhs)
            cascade_ret.append(int(K.solve_sweeps(ws.cols, lp.A.as_2d(), d, ws.inner,
                                                  ws.v_scratch, WORKERS)))
            dirs = ad.compute_directions(lp, p, backend)
            alpha = ad.step_length(p, dirs, 0.9)
            blocking.append(_blocking(p, dirs, n))
            p.x += alpha * dirs.dx
            p.y += alpha * dirs.dy
            p.s += alpha * dirs.ds
            shas.append([sha(p.x), sha(p.y), sha(p.s)])
        assert np.array_equal(p.x, q.x) and np.array_equal(p.s, q.s)
        rows = [[r.gap, r.alpha, r.primal_obj, r.dual_obj, r.r_primal, r.r_dual,
                 r.r_comp, float(r.fallback)] for r in tr]
        out[f"{tag}/A_sha"] = np.array(sha(np.asfortranarray(A).ravel(order="F")))
        out[f"{tag}/b"], out[f"{tag}/c"] = b, c
        out[f"{tag}/status"] = np.array(st.value)
        out[f"{tag}/trace"] = np.array(rows).reshape(len(rows), 8)
        out[f"{tag}/blocking"] = np.array(blocking, dtype=np.int64)
        out[f"{tag}/cascade_ret"] = np.array(cascade_ret, dtype=np.int64)
        out[f"{tag}/iter_sha"] = np.array(shas).reshape(len(shas), 3)
        out[f"{tag}/x"], out[f"{tag}/y"], out[f"{tag}/s"] = q.x, q.y, q.s
        print(tag, st.value, len(tr), "fallbacks", [int(r[7]) for r in rows],
              "cascade returns", cascade_ret)
    np.savez_compressed(os.path.join(HERE, "breakdown.npz"), **out)


def gen_check():
    """The reference's `adascale check` per seed (cli.py:183-217): the
    Woodbury and direct solutions, the backend gap and the Z-residual, for the
    default sweep (seeds 1..20, m and n drawn per seed) and a fixed 20x60 one."""
    cli = sys.modules["adascale.cli"] if "adascale.cli" in sys.modules else __import__(
        "adascale.cli", fromlist=["cli"])
    out = {}
    for tag, seeds, m, n in (("auto", range(1, 21), None, None), ("m20n60", range(1, 6), 20, 60)):
        for seed in seeds:
            rng = np.random.default_rng(seed)
            mm = m if m is not None else int(rng.integers(1, 6))
            nn = n if n is not None else int(rng.integers(mm + 1, 9))
            if mm == 1 and nn == 1:
                continue
            a, d, rhs = cli.random_system(rng, mm, nn)
            z = ad.z_inverse_check(a, d)
            wd = ad.solve_direct(a, d, rhs)
            ww = ad.solve_woodbury(ad.prepare_woodbury(a), a, d, rhs)
            gap = float(np.max(np.abs(ww - wd))) / (1.0 + float(np.max(np.abs(wd))))
            k = f"{tag}/{seed}"
            out[k + "/mn"] = np.array([mm, nn])
            out[k + "/z"], out[k + "/gap"] = np.array(z), np.array(gap)
            out[k + "/w_direct"], out[k + "/w_woodbury"] = wd, ww
            out[k + "/A"], out[k + "/d"], out[k + "/rhs"] = a.as_2d(), d, rhs
    np.savez_compressed(os.path.join(HERE, "check.npz"), **out)
    print("check.npz", len(out))


if __name__ == "__main__":
    which = sys.argv[1:] or ["kernels", "c1", "c2"]
    for w in which:
        {"kernels": gen_kernels, "c1": gen_c1, "c2": gen_c2, "c3": gen_c3, "c5": gen_c5,
         "breakdown": gen_breakdown, "check": gen_check}[w]()

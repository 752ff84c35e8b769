"""CPU oracle for the PDAS / Egidi-Maponi hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker or as the reported CPU baseline.  The product
(``paper_1502_03543_b200``) never imports it and has no CPU fallback.

Two interchangeable kernel tables, each with the reference's function table
(``adascale/_kernels.pyx`` / ``_pykernels.py``):

* ``restated()``  -- ``oracle/libpdas_oracle.so``, the plain-C restatement in
  ``oracle/pdas_oracle.c`` (always available: built by ``make -C oracle``).
* ``reference()`` -- ``oracle/_ref/_kernels*.so``, the reference's OWN compiled
  Cython core built from ``/root/reference`` by ``oracle/build_ref.sh``
  (present wherever it was built; it travels to the GPU box with the repo).

On top of a table, the solver restatement below follows ``adascale/solver.py``,
``normal.py`` and ``model.py`` line by line (cited per function), with numpy
doing the same separately-rounded elementwise arithmetic the reference does.
"""

from __future__ import annotations

import ctypes
import enum
import glob
import importlib.util
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# Constants, mirrored from the reference (cited).
DENOM_EPS_REL = 1e-12  # _kernels.pyx:21-23
SPD_EPS_REL = 1e-12  # linalg.py:17-18
SYM_TOL_REL = 1e-12  # linalg.py:19-20
FEAS_TOL_REL = 1e-8  # model.py:28
DIR_TOL_REL = 1e-8  # solver.py:24-25
GAP_TOL_REL = 1e-8  # solver.py:26-27
CAP_ALPHA = 1e6  # solver.py:28-29


# --------------------------------------------------------------------------
# kernel tables
# --------------------------------------------------------------------------

_I64 = ctypes.c_int64
_DP = ctypes.POINTER(ctypes.c_double)


def _p(a: np.ndarray):
    return a.ctypes.data_as(_DP)


class RestatedKernels:
    """numpy-level wrapper of oracle/libpdas_oracle.so with the reference table."""

    COMPILED = True
    DENOM_EPS_REL = DENOM_EPS_REL

    def __init__(self, path: Optional[str] = None):
        path = path or os.path.join(HERE, "libpdas_oracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = ctypes.CDLL(path)
        lib.or_dot_tree.argtypes = [_DP, _I64, _DP, _I64, _I64, _DP]
        lib.or_mat_vec.argtypes = [_DP, _I64, _I64, _DP, _DP]
        lib.or_mat_t_vec.argtypes = [_DP, _I64, _I64, _DP, _DP]
        lib.or_gram.argtypes = [_DP, _I64, _I64, ctypes.c_void_p, _DP]
        lib.or_cholesky_factor.argtypes = [_DP, _I64, ctypes.c_double, _DP]
        lib.or_cholesky_factor.restype = _I64
        lib.or_cholesky_solve_many.argtypes = [_DP, _I64, _DP, _I64]
        lib.or_build_v.argtypes = [_DP, _I64, _I64, ctypes.c_double, _DP]
        lib.or_sweep_phase1.argtypes = [_DP, _I64, _DP, _DP, _I64, _I64]
        lib.or_sweep_phase2.argtypes = [_DP, _I64, _I64, _DP, ctypes.c_double, _I64, _I64]
        lib.or_solve_sweeps.argtypes = [_DP, _DP, _DP, _DP, _DP, _I64, _I64, ctypes.c_int]
        lib.or_solve_sweeps.restype = ctypes.c_int
        lib.or_solve_sweeps_prefix.argtypes = [_DP, _DP, _DP, _DP, _DP, _I64, _I64, _I64, ctypes.c_int]
        lib.or_solve_sweeps_prefix.restype = ctypes.c_int
        self.lib = lib

    @staticmethod
    def _f(a):
        a = np.asarray(a)
        if a.dtype != np.float64 or not a.flags.f_contiguous:
            raise ValueError("expected F-contiguous float64")
        return a

    @staticmethod
    def _c(a):
        a = np.asarray(a)
        if a.dtype != np.float64 or not a.flags.c_contiguous or a.ndim != 1:
            raise ValueError("expected contiguous float64 vector")
        return a

    def dot_tree(self, u, v):
        u = np.asarray(u, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        out = ctypes.c_double()
        su, sv = u.strides[0] // 8, v.strides[0] // 8
        self.lib.or_dot_tree(
            ctypes.cast(u.ctypes.data, _DP), su, ctypes.cast(v.ctypes.data, _DP), sv,
            u.shape[0], ctypes.byref(out))
        return out.value

    def mat_vec(self, a, x):
        a, x = self._f(a), self._c(x)
        out = np.empty(a.shape[0])
        self.lib.or_mat_vec(_p(a), a.shape[0], a.shape[1], _p(x), _p(out))
        return out

    def mat_t_vec(self, a, y):
        a, y = self._f(a), self._c(y)
        out = np.empty(a.shape[1])
        self.lib.or_mat_t_vec(_p(a), a.shape[0], a.shape[1], _p(y), _p(out))
        return out

    def gram(self, a):
        a = self._f(a)
        g = np.zeros((a.shape[0], a.shape[0]), order="F")
        self.lib.or_gram(_p(a), a.shape[0], a.shape[1], None, _p(g))
        return g

    def scaled_gram(self, a, d):
        a, d = self._f(a), self._c(d)
        g = np.zeros((a.shape[0], a.shape[0]), order="F")
        self.lib.or_gram(_p(a), a.shape[0], a.shape[1], d.ctypes.data, _p(g))
        return g

    def cholesky_factor(self, g, eps_rel):
        g = self._f(g)
        low = np.zeros_like(g, order="F")
        fail = self.lib.or_cholesky_factor(_p(g), g.shape[0], eps_rel, _p(low))
        return low, int(fail)

    def cholesky_solve_many(self, low, b):
        low = self._f(low)
        x = np.array(b, dtype=np.float64, order="F", copy=True)
        self.lib.or_cholesky_solve_many(_p(low), low.shape[0], _p(x), x.shape[1])
        return x

    def build_v(self, a, l0, dl, v):
        a = self._f(a)
        self.lib.or_build_v(_p(a), a.shape[0], l0, dl, _p(self._c(v)))

    def sweep_phase1(self, cols, v, inner, k0, k1):
        cols = self._f(cols)
        self.lib.or_sweep_phase1(_p(cols), cols.shape[0], _p(self._c(v)), _p(self._c(inner)), k0, k1)

    def sweep_phase2(self, cols, l0, inner, denom, k0, k1):
        cols = self._f(cols)
        self.lib.or_sweep_phase2(_p(cols), cols.shape[0], l0, _p(self._c(inner)), denom, k0, k1)

    def solve_sweeps(self, cols, a, d, inner, v, workers):
        cols, a = self._f(cols), self._f(a)
        return int(self.lib.or_solve_sweeps(
            _p(cols), _p(a), _p(self._c(d)), _p(self._c(inner)), _p(self._c(v)),
            a.shape[0], a.shape[1], int(workers)))

    def solve_sweeps_prefix(self, cols, a, d, inner, v, steps, workers):
        cols, a = self._f(cols), self._f(a)
        return int(self.lib.or_solve_sweeps_prefix(
            _p(cols), _p(a), _p(self._c(d)), _p(self._c(inner)), _p(self._c(v)),
            a.shape[0], a.shape[1], int(steps), int(workers)))


_RESTATED = None
_REFERENCE = None


def restated() -> RestatedKernels:
    global _RESTATED
    if _RESTATED is None:
        _RESTATED = RestatedKernels()
    return _RESTATED


def reference_path() -> Optional[str]:
    hits = sorted(glob.glob(os.path.join(HERE, "_ref", "_kernels*.so")))
    return hits[0] if hits else None


def reference():
    """The reference's own compiled core (oracle/_ref), or None if not built."""
    global _REFERENCE
    if _REFERENCE is None:
        path = reference_path()
        if path is None:
            return None
        spec = importlib.util.spec_from_file_location("adascale._kernels", path)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REFERENCE = mod
    return _REFERENCE


def best():
    """Reference core when built, else the restatement (both are bitwise equal)."""
    return reference() or restated()


# --------------------------------------------------------------------------
# solver restatement (adascale/{model,normal,solver}.py)
# --------------------------------------------------------------------------


class OracleError(Exception):
    pass


class NotPositiveDefinite(OracleError):
    pass


class SingularUpdate(OracleError):
    pass


class NotInterior(OracleError):
    pass


class Status(enum.Enum):  # solver.py:34-38
    OPTIMAL = "optimal"
    ITER_LIMIT = "iter_limit"
    UNBOUNDED = "unbounded"
    NUMERICAL_BREAKDOWN = "numerical_breakdown"


def _fortran(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def cholesky(k, g):
    """linalg.py:107-123 (symmetry check, kernel call, fail -> exception)."""
    g = _fortran(g)
    scale = float(np.max(np.abs(g))) if g.size else 0.0
    if g.size and float(np.max(np.abs(g - g.T))) > SYM_TOL_REL * max(scale, 1.0):
        raise ValueError("cholesky_factor requires a symmetric matrix")
    low, fail = k.cholesky_factor(g, SPD_EPS_REL)
    if fail >= 0:
        raise NotPositiveDefinite(f"nonpositive pivot at column {fail}")
    return np.asarray(low)


def cholesky_solve(k, low, b):
    """linalg.py:126-132."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = k.cholesky_solve_many(low, b.reshape((-1, 1), order="F"))
    return np.ascontiguousarray(np.asarray(x).ravel(order="F"))


def gen_random_feasible(k, m: int, n: int, seed: int):
    """model.py:134-161.  Returns (A F-order, b, c, x, y, s)."""
    if not 1 <= m < n:
        raise ValueError(f"generator requires 1 <= m < n, got m={m}, n={n}")
    rng = np.random.default_rng(seed)
    a = None
    for _ in range(100):
        cand = _fortran(rng.uniform(-1.0, 1.0, size=(m, n)))
        try:
            cholesky(k, k.gram(cand))
        except NotPositiveDefinite:
            continue
        a = cand
        break
    if a is None:
        raise OracleError("no full-rank draw")
    x = rng.uniform(0.5, 2.0, size=n)
    s = rng.uniform(0.5, 2.0, size=n)
    y = rng.uniform(-1.0, 1.0, size=m)
    b = np.asarray(k.mat_vec(a, x))
    c = np.asarray(k.mat_t_vec(a, y)) + s
    return a, b, c, x, y, s


def random_system(k, rng, m: int, n: int):
    """cli.py:165-180: full-rank A, d = 10**U[-3,3], rhs ~ U[-1,1]."""
    a = None
    for _ in range(100):
        cand = _fortran(rng.uniform(-1.0, 1.0, size=(m, n)))
        try:
            cholesky(k, k.gram(cand))
        except NotPositiveDefinite:
            continue
        a = cand
        break
    d = np.power(10.0, rng.uniform(-3.0, 3.0, size=n))
    rhs = rng.uniform(-1.0, 1.0, size=m)
    return a, d, rhs


@dataclass
class Basis:  # normal.py:38-51
    L0: np.ndarray
    Y: np.ndarray


def prepare_woodbury(k, a) -> Basis:
    """normal.py:108-112."""
    low = cholesky(k, k.gram(a))
    y = np.asfortranarray(k.cholesky_solve_many(low, a))
    return Basis(low, y)


def init_workspace(k, basis: Basis, rhs):
    """normal.py:115-124: cols = [Y | (AA^T)^{-1} rhs]."""
    m, n = basis.Y.shape
    cols = np.zeros((m, n + 1), dtype=np.float64, order="F")
    cols[:, :n] = basis.Y
    cols[:, n] = cholesky_solve(k, basis.L0, rhs)
    return cols, np.zeros(n + 1), np.zeros(m)


def solve_woodbury(k, basis: Basis, a, d, rhs, workers: int = 1):
    """normal.py:163-175."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    if d.size and float(np.min(d)) <= 0.0:
        raise ValueError("solve_woodbury requires strictly positive scaling entries")
    cols, inner, v = init_workspace(k, basis, rhs)
    fail = k.solve_sweeps(cols, a, d, inner, v, workers)
    if fail:
        raise SingularUpdate(f"update denominator vanished at step {fail}")
    return cols[:, -1].copy()


def solve_direct(k, a, d, rhs):
    """normal.py:101-105."""
    low = cholesky(k, k.scaled_gram(a, np.ascontiguousarray(d, dtype=np.float64)))
    return cholesky_solve(k, low, rhs)


@dataclass
class Dirs:  # solver.py:41-51
    dx: np.ndarray
    dy: np.ndarray
    ds: np.ndarray
    residual_primal: float
    residual_dual: float
    residual_comp: float
    fallback: bool = False


@dataclass
class Trace:  # solver.py:75-86
    iter: int
    gap: float
    alpha: float
    primal_obj: float
    dual_obj: float
    r_primal: float
    r_dual: float
    r_comp: float
    millis: float
    fallback: bool = False
    blocking: int = -1  # extra: argmin index of the ratio test (-1: none)


def compute_directions(k, a, x, s, solve):
    """solver.py:152-172 (scaling_diag :142-145 included)."""
    if x.size == 0 or float(np.min(x)) <= 0.0 or float(np.min(s)) <= 0.0:
        raise NotInterior("point is not strictly interior")
    d = x / s
    rhs = np.asarray(k.mat_vec(a, x))
    fallback = False
    try:
        dy = solve(d, rhs)
    except SingularUpdate:
        dy = solve_direct(k, a, d, rhs)
        fallback = True
    t = np.asarray(k.mat_t_vec(a, dy))
    ds = -t
    dx = d * t - x
    r_primal = float(np.max(np.abs(np.asarray(k.mat_vec(a, dx)))))
    r_dual = float(np.max(np.abs(ds + t)))
    r_comp = float(np.max(np.abs(s * dx + x * ds + x * s)))
    return Dirs(dx, dy, ds, r_primal, r_dual, r_comp, fallback)


def step_length(x, s, dirs: Dirs, rho: float):
    """solver.py:175-189; also returns the blocking index (argmin over the
    concatenation [x-ratios (index j), s-ratios (index n+j)], first minimum)."""
    n = x.size
    ratios = []
    best_idx = -1
    best_val = None
    neg = dirs.dx < 0.0
    if neg.any():
        r = -x[neg] / dirs.dx[neg]
        j = int(np.argmin(r))
        ratios.append(float(r[j]))
        best_val, best_idx = float(r[j]), int(np.nonzero(neg)[0][j])
    neg = dirs.ds < 0.0
    if neg.any():
        r = -s[neg] / dirs.ds[neg]
        j = int(np.argmin(r))
        ratios.append(float(r[j]))
        if best_val is None or float(r[j]) < best_val:
            best_val, best_idx = float(r[j]), n + int(np.nonzero(neg)[0][j])
    if not ratios:
        return CAP_ALPHA, -1
    return rho * min(ratios), best_idx


def solve_lp(k, a, b, c, x, y, s, rho=0.9, gap_tol=None, max_iter=500, backend="woodbury",
             workers=1, basis: Optional[Basis] = None, on_iter=None):
    """solver.py:197-279.  Returns (x, y, s, Status, [Trace])."""
    a = _fortran(a)
    cholesky(k, k.gram(a))  # validate (model.py:87-102): rank certificate
    x, y, s = (np.array(v, dtype=np.float64, copy=True) for v in (x, y, s))
    if x.size == 0 or float(np.min(x)) <= 0.0 or float(np.min(s)) <= 0.0:
        raise NotInterior("start is not strictly interior")
    if backend == "woodbury":
        basis = basis or prepare_woodbury(k, a)
        solve = lambda d, rhs: solve_woodbury(k, basis, a, d, rhs, workers)  # noqa: E731
    else:
        solve = lambda d, rhs: solve_direct(k, a, d, rhs)  # noqa: E731
    gap = k.dot_tree(x, s)
    if gap_tol is None:
        gap_tol = GAP_TOL_REL * (1.0 + abs(k.dot_tree(c, x)))
    trace: List[Trace] = []
    if gap <= gap_tol:
        return x, y, s, Status.OPTIMAL, trace
    status = Status.ITER_LIMIT
    for it in range(1, max_iter + 1):
        t0 = time.perf_counter()
        try:
            dirs = compute_directions(k, a, x, s, solve)
        except (NotPositiveDefinite, SingularUpdate):
            status = Status.NUMERICAL_BREAKDOWN
            break
        if not (np.isfinite(dirs.dx).all() and np.isfinite(dirs.dy).all()
                and np.isfinite(dirs.ds).all()):
            status = Status.NUMERICAL_BREAKDOWN
            break
        alpha, blocking = step_length(x, s, dirs, rho)
        if alpha >= CAP_ALPHA:
            millis = (time.perf_counter() - t0) * 1e3
            trace.append(Trace(it, gap, alpha, k.dot_tree(c, x), k.dot_tree(b, y),
                               dirs.residual_primal, dirs.residual_dual, dirs.residual_comp,
                               millis, dirs.fallback, blocking))
            status = Status.UNBOUNDED
            break
        x += alpha * dirs.dx
        y += alpha * dirs.dy
        s += alpha * dirs.ds
        gap = k.dot_tree(x, s)
        millis = (time.perf_counter() - t0) * 1e3
        trace.append(Trace(it, gap, alpha, k.dot_tree(c, x), k.dot_tree(b, y),
                           dirs.residual_primal, dirs.residual_dual, dirs.residual_comp,
                           millis, dirs.fallback, blocking))
        if on_iter is not None:
            on_iter(it, x, y, s, dirs)
        if gap <= gap_tol:
            status = Status.OPTIMAL
            break
    return x, y, s, status, trace

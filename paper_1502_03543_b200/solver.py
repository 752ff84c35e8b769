"""Primal-dual affine scaling driver -- the drop-in `solve_lp`.

Mirrors adascale/solver.py: Status (:34-38), Directions (:41-51),
SolveOptions (:54-72), TraceRecord (:75-86), the trace writers (:89-103),
the backends (:106-139), scaling_diag (:142-145), compute_directions
(:152-172), step_length (:175-189), duality_gap (:192-194), solve_lp
(:197-279) and z_inverse_check (:282-315).  Same signatures, constants,
exceptions, status semantics and trace layout.

`solve_lp` keeps the whole iteration device-resident (engine.DeviceSolver):
per iteration only the PdasIterState block (scalars) comes back to the host,
where the termination logic of solver.py:222-278 runs unchanged.
"""

from __future__ import annotations

import enum
import json
import time
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

from . import _device as dv
from .engine import DeviceProblem, DeviceSolver, d_mat_t_vec, d_mat_vec, not_interior
from .errors import NotInterior, NotPositiveDefinite, SingularUpdate
from .linalg import DenseMatrix, as_vector, cholesky_factor, cholesky_solve_many, dot_tree, scaled_gram
from .model import InteriorPoint, StandardFormLP, check_interior, feas_tol
from .normal import solve_direct
from .parallel import resolve_workers

DIR_TOL_REL = 1e-8  # direction residual certification, relative to 1 + |x|_inf |s|_inf
GAP_TOL_REL = 1e-8  # default stopping gap, relative to 1 + |c'x0|
CAP_ALPHA = 1e6  # step returned when no component blocks (likely unbounded ray)

BACKENDS = ("direct", "woodbury")


class Status(enum.Enum):
    OPTIMAL = "optimal"
    ITER_LIMIT = "iter_limit"
    UNBOUNDED = "unbounded"
    NUMERICAL_BREAKDOWN = "numerical_breakdown"


@dataclass(eq=False)
class Directions:
    """Affine-scaling step (dx, dy, ds) with its residual certificates."""

    dx: np.ndarray
    dy: np.ndarray
    ds: np.ndarray
    residual_primal: float
    residual_dual: float
    residual_comp: float
    fallback: bool = False


@dataclass
class SolveOptions:
    rho: float = 0.9
    gap_tol: Optional[float] = None
    max_iter: int = 500
    backend: str = "woodbury"
    workers: int = 1

    def __post_init__(self):
        if not 0.0 < self.rho < 1.0:
            raise ValueError("rho must be in (0,1)")
        if self.gap_tol is not None and not self.gap_tol > 0.0:
            raise ValueError("gap-tol must be positive")
        if self.max_iter < 1:
            raise ValueError("max-iter must be >= 1")
        if self.backend not in BACKENDS:
            raise ValueError(f"backend must be one of {', '.join(BACKENDS)}")
        if self.workers < 0:
            raise ValueError("workers must be >= 0")


@dataclass
class TraceRecord:
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


TRACE_CSV_HEADER = "iter,gap,alpha,primal_obj,dual_obj,r_primal,r_dual,r_comp,millis"


def trace_to_csv(trace: List[TraceRecord]) -> str:
    lines = [TRACE_CSV_HEADER]
    for r in trace:
        lines.append(f"{r.iter},{r.gap!r},{r.alpha!r},{r.primal_obj!r},{r.dual_obj!r},"
                     f"{r.r_primal!r},{r.r_dual!r},{r.r_comp!r},{r.millis!r}")
    return "\n".join(lines) + "\n"


def trace_to_json(trace: List[TraceRecord]) -> str:
    return json.dumps([vars(r) for r in trace])


# ------------------------------------------------------------------ backends
class _DeviceBackend:
    name = "?"

    def __init__(self, lp: StandardFormLP, backend: str, workers: int = 1):
        self.lp = lp
        self.workers = resolve_workers(workers)
        self.prob = DeviceProblem.from_lp(lp)
        self.engine = DeviceSolver(self.prob, backend)

    def solve(self, d, rhs) -> np.ndarray:
        """dy for (A diag(d) A^T) dy = rhs; SingularUpdate on breakdown."""
        eng = self.engine
        eng.d.copy_(dv.torch().from_numpy(as_vector(d, "d")))
        eng.rhs.copy_(dv.torch().from_numpy(as_vector(rhs, "rhs")))
        st = dv.stream()
        from ._lib import OFF_CASCADE_FAIL, OFF_CHOL_FAIL, call

        call("pdas_iter_reset", eng._sptr(), st)
        if eng.backend == "woodbury":
            if float(np.min(d)) <= 0.0:
                raise ValueError("solve_woodbury requires strictly positive scaling entries")
            m, n = eng.m, eng.n
            eng.cols[:m * n].copy_(eng.basis.Y)
            eng.xcol.copy_(eng.rhs)
            call("pdas_cholesky_solve_many", dv.ptr(eng.basis.L0), m, dv.ptr(eng.xcol), 1, st)
            call("pdas_solve_sweeps", dv.ptr(eng.cols), dv.ptr(eng.prob.A), dv.ptr(eng.d), None,
                 None, m, n, 1, eng._sptr(OFF_CASCADE_FAIL), st)
            s = eng._fetch_state()
            if s.cascade_fail:
                raise SingularUpdate(f"update denominator vanished at step {s.cascade_fail}")
            return dv.download(eng.xcol)
        eng._solve_direct_into(eng.dy_direct, eng._sptr(OFF_CHOL_FAIL))
        s = eng._fetch_state()
        if s.chol_fail >= 0:
            raise NotPositiveDefinite(f"nonpositive pivot at column {s.chol_fail}")
        return dv.download(eng.dy_direct)


class DirectBackend(_DeviceBackend):
    """Fresh Cholesky factorisation of A diag(d) A^T per solve."""

    name = "direct"

    def __init__(self, lp: StandardFormLP):
        super().__init__(lp, "direct")


class WoodburyBackend(_DeviceBackend):
    """Rank-one-update cascade over a basis factored once per problem."""

    name = "woodbury"

    def __init__(self, lp: StandardFormLP, workers: int = 1):
        super().__init__(lp, "woodbury", workers)


def make_backend(lp: StandardFormLP, name: str, workers: int = 1):
    if name == "direct":
        return DirectBackend(lp)
    if name == "woodbury":
        return WoodburyBackend(lp, workers)
    raise ValueError(f"backend must be one of {', '.join(BACKENDS)}")


# ------------------------------------------------------------------ pieces
def _state_scratch():
    t = dv.require_gpu()
    from ._lib import STATE_BYTES, call

    state = t.zeros(STATE_BYTES, dtype=t.uint8, device=dv.device())
    call("pdas_iter_reset", dv.ptr(state), dv.stream())
    return state


def _fetch(state):
    from ._lib import PdasIterState

    return PdasIterState.from_buffer_copy(dv.download(state).tobytes())


def scaling_diag(p: InteriorPoint) -> np.ndarray:
    """d = x/s, the only iteration-dependent part of the normal equations
    (solver.py:142-145; the engine's k_scaling kernel)."""
    check_interior(p)
    from ._lib import call

    x, s = dv.upload(p.x), dv.upload(p.s)
    d = dv.empty(p.x.size)
    call("pdas_iter_scaling", dv.ptr(x), dv.ptr(s), p.x.size, dv.ptr(d),
         dv.ptr(_state_scratch()), dv.stream())
    return dv.download(d)


def dir_tol(p: InteriorPoint) -> float:
    return DIR_TOL_REL * (1.0 + float(np.max(np.abs(p.x))) * float(np.max(np.abs(p.s))))


def compute_directions(lp: StandardFormLP, p: InteriorPoint, backend) -> Directions:
    """Closed-form affine-scaling directions (solver.py:152-172), on device.
    A SingularUpdate in the cascade retries with the direct solve, flagged."""
    eng = backend.engine if isinstance(backend, _DeviceBackend) else make_backend(
        lp, getattr(backend, "name", "woodbury")).engine
    eng.load_iterate(p.x, p.y, p.s)
    eng.enqueue_solve()
    from ._lib import call

    st = dv.stream()
    call("pdas_iter_directions", dv.ptr(eng.prob.A), eng.m, eng.n, dv.ptr(eng.dy), dv.ptr(eng.d),
         dv.ptr(eng.x), dv.ptr(eng.s), dv.ptr(eng.dx), dv.ptr(eng.ds), 0.9, eng._sptr(), st)
    s = eng._fetch_state()
    if not_interior(s.interior_flags):
        raise NotInterior("point is not strictly interior (needs x > 0 and s > 0)")
    fallback = False
    if eng.backend == "woodbury" and s.cascade_fail:
        from ._lib import OFF_CASCADE_FAIL, OFF_CHOL_FAIL

        eng.state[OFF_CASCADE_FAIL:OFF_CASCADE_FAIL + 4].zero_()
        eng._solve_direct_into(eng.dy_direct, eng._sptr(OFF_CHOL_FAIL))
        eng.dy = eng.dy_direct
        call("pdas_iter_directions", dv.ptr(eng.prob.A), eng.m, eng.n, dv.ptr(eng.dy),
             dv.ptr(eng.d), dv.ptr(eng.x), dv.ptr(eng.s), dv.ptr(eng.dx), dv.ptr(eng.ds), 0.9,
             eng._sptr(), st)
        s = eng._fetch_state()
        fallback = True
    if s.chol_fail >= 0:
        raise NotPositiveDefinite(f"nonpositive pivot at column {s.chol_fail}")
    return Directions(dv.download(eng.dx), dv.download(eng.dy), dv.download(eng.ds),
                      s.r_primal, s.r_dual, s.r_comp, fallback)


def step_length(p: InteriorPoint, dirs: Directions, rho: float) -> float:
    """rho times the largest interior-preserving step; CAP_ALPHA when nothing
    blocks (solver.py:175-189).  The engine's ratio test (pdas_ratio_test)."""
    from ._lib import call

    n = p.x.size
    x, s = dv.upload(p.x), dv.upload(p.s)
    dx, ds = dv.upload(dirs.dx), dv.upload(dirs.ds)
    state = _state_scratch()
    call("pdas_ratio_test", dv.ptr(x), dv.ptr(s), dv.ptr(dx), dv.ptr(ds), n, float(rho),
         dv.ptr(state), dv.stream())
    return float(_fetch(state).alpha)


def duality_gap(p: InteriorPoint) -> float:
    """x's (tree order), zero at optimality for feasible pairs."""
    return dot_tree(p.x, p.s)


# ------------------------------------------------------------------ solve_lp
def _check_feasible_device(lp: StandardFormLP, prob: DeviceProblem, p: InteriorPoint) -> None:
    """model.py:122-131 evaluated against the device-resident problem."""
    from .errors import DimensionMismatch, NotFeasible

    if p.x.size != lp.n or p.s.size != lp.n or p.y.size != lp.m:
        raise DimensionMismatch("point dimensions do not match the problem")
    t = dv.require_gpu()
    tol = feas_tol(lp)
    x, y, s = dv.upload(p.x), dv.upload(p.y), dv.upload(p.s)
    rp = float(t.max(t.abs(t.sub(d_mat_vec(prob.A, prob.m, prob.n, x), prob.b))).item())
    atv = d_mat_t_vec(prob.A, prob.m, prob.n, y)
    rd = float(t.max(t.abs(t.sub(s, t.sub(prob.c, atv)))).item())
    if rp > tol or rd > tol:
        raise NotFeasible(
            f"start violates feasibility: primal {rp:.3e}, dual {rd:.3e}, tol {tol:.3e}")


def solve_lp(
    lp: StandardFormLP,
    start: InteriorPoint,
    opts: Optional[SolveOptions] = None,
    *,
    group=None,
    exchange: str = "nccl",
) -> Tuple[InteriorPoint, Status, List[TraceRecord]]:
    """Run the affine-scaling iteration from a strictly feasible start.

    Returns the final iterate, a termination status and one trace record per
    completed iteration (solver.py:197-279).  Backend failures that survive
    the direct fallback surface as NUMERICAL_BREAKDOWN with the partial trace.

    group: a torch.distributed process group (one process per GPU, every rank
    calling with the same problem): the Woodbury cascade then runs
    column-sharded over the group (dist.py); results are bitwise the 1-GPU
    ones on every rank.  exchange: "nccl" (one broadcast per pivot block) or
    "peer" (EXPERIMENTAL: the panel stores finished blocks straight into the
    peers' buffers over NVLink, torch symmetric memory; dist.ShardedSolver --
    not yet run on two real GPUs).
    """
    opts = opts or SolveOptions()
    prob = DeviceProblem.from_lp(lp)
    L0 = prob.validate()  # NonFiniteEntry / RankDeficient (model.py:87-102)
    p = start.copy()
    check_interior(p)
    _check_feasible_device(lp, prob, p)
    resolve_workers(opts.workers)
    if group is not None and opts.backend == "woodbury":
        from .dist import ShardedSolver

        eng = ShardedSolver(prob, group, opts.rho, L0=L0, exchange=exchange)
    else:
        eng = DeviceSolver(prob, opts.backend, opts.rho,
                           L0=L0 if opts.backend == "woodbury" else None)
    eng.load_iterate(p.x, p.y, p.s)
    st0 = eng.objectives()
    gap = st0.gap
    gap_tol = opts.gap_tol
    if gap_tol is None:
        gap_tol = GAP_TOL_REL * (1.0 + abs(st0.pobj))
    trace: List[TraceRecord] = []
    if gap <= gap_tol:
        return p, Status.OPTIMAL, trace
    status = Status.ITER_LIMIT
    for it in range(1, opts.max_iter + 1):
        res = eng.iterate()
        st = res.state
        if not_interior(st.interior_flags):
            raise NotInterior("point is not strictly interior (needs x > 0 and s > 0)")
        if st.chol_fail >= 0:  # NotPositiveDefinite in the direct solve / fallback
            status = Status.NUMERICAL_BREAKDOWN
            break
        if st.nonfinite:
            status = Status.NUMERICAL_BREAKDOWN
            break
        rec = TraceRecord(it, gap, st.alpha, st.pobj, st.dobj, st.r_primal, st.r_dual,
                          st.r_comp, res.millis, bool(st.fallback))
        if st.alpha >= CAP_ALPHA:
            trace.append(rec)
            status = Status.UNBOUNDED
            break
        gap = st.gap
        rec.gap = gap
        trace.append(rec)
        if gap <= gap_tol:
            status = Status.OPTIMAL
            break
    x, y, s = eng.read_iterate()
    return InteriorPoint(x, y, s), status, trace


def z_inverse_check(a: DenseMatrix, d) -> float:
    """|Z Zhat^{-1} - I|_max for the blockwise inverse of
    Z = [[0, A', I], [A, 0, 0], [I, 0, diag(d)]] (solver.py:282-315).
    Verification utility; dense fp64 products on the GPU."""
    t = dv.require_gpu()
    dev = dv.device()
    m, n = a.rows, a.cols
    d = np.ascontiguousarray(d, dtype=np.float64)
    low = cholesky_factor(scaled_gram(a, d))
    x_inv = t.from_numpy(np.asarray(cholesky_solve_many(low, np.eye(m)))).to(dev)
    a2 = t.from_numpy(np.ascontiguousarray(a.as_2d())).to(dev)
    dd = t.from_numpy(d).to(dev)
    xa = x_inv @ a2
    dat = dd[:, None] * a2.T
    dat_x = dat @ x_inv
    dat_xa = dat @ xa
    eye_n = t.eye(n, dtype=t.float64, device=dev)
    b13 = eye_n - dat_xa
    z = t.cat([
        t.cat([t.zeros(n, n, dtype=t.float64, device=dev), a2.T, eye_n], 1),
        t.cat([a2, t.zeros(m, m, dtype=t.float64, device=dev),
               t.zeros(m, n, dtype=t.float64, device=dev)], 1),
        t.cat([eye_n, t.zeros(n, m, dtype=t.float64, device=dev), t.diag(dd)], 1),
    ], 0)
    z_inv = t.cat([
        t.cat([dat_xa * dd[None, :] - t.diag(dd), dat_x, b13], 1),
        t.cat([xa * dd[None, :], x_inv, -xa], 1),
        t.cat([b13.T, -(a2.T @ x_inv), a2.T @ xa], 1),
    ], 0)
    dim = 2 * n + m
    return float(t.max(t.abs(z @ z_inv - t.eye(dim, dtype=t.float64, device=dev))).item())


__all__ = [
    "BACKENDS", "CAP_ALPHA", "DIR_TOL_REL", "GAP_TOL_REL", "DirectBackend", "Directions",
    "SolveOptions", "Status", "TraceRecord", "WoodburyBackend", "compute_directions",
    "dir_tol", "duality_gap", "make_backend", "scaling_diag", "solve_direct", "solve_lp",
    "step_length", "trace_to_csv", "trace_to_json", "z_inverse_check", "SingularUpdate",
]

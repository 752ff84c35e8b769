"""Device-resident PDAS engine: the hot path behind `solve_lp`.

One `DeviceSolver` owns, on one GPU:
  * the problem  A (m x n, column-major), b, c                 (model.py:33-62)
  * the Woodbury basis L0 = chol(A A^T), Y = (A A^T)^{-1} A    (normal.py:38-51, 108-112)
  * the augmented workspace [Y | x] (m x (n+1))                (normal.py:54-88, 115-124)
  * the iterate x, y, s and the direction vectors dx, dy, ds
  * a PdasIterState block the kernels fill in every iteration.

`iterate()` enqueues one full PDAS iteration (solver.py:222-278) on the
current stream -- scaling, A x, x0 = L0^-T L0^-1 (A x), the rank-one cascade,
A^T dy, residuals, ratio test, the x/y/s update, gap and objectives -- then
copies the state block back once and synchronises.  Only scalars cross the
PCIe bus per iteration; the SingularUpdate fallback to the direct solve
(solver.py:161-165) is decided on the host from that state and re-enqueued.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import _device as dv
from ._lib import (
    load,
    OFF_CASCADE_FAIL,
    OFF_CHOL_FAIL,
    STATE_BYTES,
    PdasIterState,
    call,
)
from .errors import NonFiniteEntry, NotPositiveDefinite, RankDeficient
from .linalg import SPD_EPS_REL

IT_X_NAN, IT_X_LE0, IT_S_NAN, IT_S_LE0 = 1, 2, 4, 8


def not_interior(flags: int) -> bool:
    """model.py:116-119 under np.min semantics (a NaN makes the min NaN)."""
    return bool(((flags & IT_X_LE0) and not (flags & IT_X_NAN))
                or ((flags & IT_S_LE0) and not (flags & IT_S_NAN)))


# ----------------------------------------------------------- device primitives
def d_mat_vec(A, m, n, x, out=None):
    out = dv.empty(m) if out is None else out
    call("pdas_mat_vec", dv.ptr(A), m, n, dv.ptr(x), dv.ptr(out), dv.stream())
    return out


def d_mat_t_vec(A, m, n, y, out=None):
    out = dv.empty(n) if out is None else out
    call("pdas_mat_t_vec", dv.ptr(A), m, n, dv.ptr(y), dv.ptr(out), dv.stream())
    return out


def d_gram(A, m, n, d=None):
    g = dv.empty(m * m)
    if d is None:
        call("pdas_gram", dv.ptr(A), m, n, dv.ptr(g), dv.stream())
    else:
        call("pdas_scaled_gram", dv.ptr(A), m, n, dv.ptr(d), dv.ptr(g), dv.stream())
    return g


def d_cholesky(G, nn, fail_ptr=None):
    """Factor on device; returns (L, fail_tensor).  fail_ptr: write the fail
    column to that device address instead (e.g. inside the iteration state)."""
    t = dv.torch()
    L = dv.empty(nn * nn)
    fail = None
    if fail_ptr is None:
        fail = dv.empty(1, dtype=t.int64)
        fail_ptr = dv.ptr(fail)
    call("pdas_cholesky_factor", dv.ptr(G), nn, SPD_EPS_REL, dv.ptr(L), fail_ptr, dv.stream())
    return L, fail


def d_solve_many(L, m, X, k):
    call("pdas_cholesky_solve_many", dv.ptr(L), m, dv.ptr(X), k, dv.stream())
    return X


def d_dot(u, v):
    out = dv.empty(1)
    call("pdas_dot_tree", dv.ptr(u), 1, dv.ptr(v), 1, u.numel(), dv.ptr(out), dv.stream())
    return out


# ----------------------------------------------------------- problem + basis
class DeviceProblem:
    """A, b, c resident on the current device."""

    def __init__(self, A2d_or_flat, b, c, m: int, n: int):
        self.m, self.n = int(m), int(n)
        a = np.asarray(A2d_or_flat, dtype=np.float64)
        self.A = dv.upload(a if a.ndim == 2 else a.reshape((m, n), order="F"))
        self.b = dv.upload(b)
        self.c = dv.upload(c)

    @classmethod
    def from_lp(cls, lp) -> "DeviceProblem":
        return cls(lp.A.data, lp.b, lp.c, lp.m, lp.n)

    def validate(self):
        """model.py:87-102: finiteness, then full row rank via chol(A A^T).
        Returns the factor so prepare() need not recompute it."""
        t = dv.torch()
        for name, v in (("A", self.A), ("b", self.b), ("c", self.c)):
            if not bool(t.isfinite(v).all()):
                raise NonFiniteEntry(f"{name} contains a non-finite entry")
        L0, fail = d_cholesky(d_gram(self.A, self.m, self.n), self.m)
        f = int(fail.item())
        if f >= 0:
            raise RankDeficient(
                f"A does not have full row rank: nonpositive pivot at column {f}")
        return L0


class DeviceBasis:
    """Iteration-invariant L0 and Y (normal.py:38-51) on device."""

    def __init__(self, L0, Y, m: int, n: int):
        self.L0, self.Y, self.m, self.n = L0, Y, m, n


def prepare_basis(prob: DeviceProblem, L0=None) -> DeviceBasis:
    """normal.py:108-112: L0 = chol(gram(A)); Y = L0^-T L0^-1 A."""
    m, n = prob.m, prob.n
    if L0 is None:
        L0, fail = d_cholesky(d_gram(prob.A, m, n), m)
        f = int(fail.item())
        if f >= 0:
            raise NotPositiveDefinite(f"nonpositive pivot at column {f}")
    Y = prob.A.clone()
    d_solve_many(L0, m, Y, n)
    return DeviceBasis(L0, Y, m, n)


# ----------------------------------------------------------- solver engine
class IterResult:
    """Host view of one iteration's PdasIterState."""

    __slots__ = ("state", "millis")

    def __init__(self, state: PdasIterState, millis: float):
        self.state = state
        self.millis = millis

    def __getattr__(self, k):
        return getattr(self.state, k)


class DeviceSolver:
    """Device-resident PDAS iteration for one LP (see module docstring)."""

    # subclasses whose iteration is not one replayable launch sequence (the
    # sharded solver: collectives, per-rank schedule) turn the graph off
    graph_iterations = True

    def __init__(self, prob: DeviceProblem, backend: str = "woodbury", rho: float = 0.9,
                 basis: DeviceBasis = None, L0=None):
        t = dv.require_gpu()
        self.t = t
        self.prob = prob
        self.backend = backend
        self.rho = float(rho)
        m, n = prob.m, prob.n
        self.m, self.n = m, n
        self.basis = None
        if backend == "woodbury":
            self.basis = basis or prepare_basis(prob, L0)
            self.cols = dv.empty(m * (n + 1))
            self.casc_ws = t.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=t.uint8,
                                   device=dv.device())
            self.epoch = 0
            self.xcol = self.cols[m * n:]
        self.x = dv.empty(n)
        self.y = dv.empty(m)
        self.s = dv.empty(n)
        self.d = dv.empty(n)
        self.rhs = dv.empty(m)
        self.dx = dv.empty(n)
        self.ds = dv.empty(n)
        self.dy_direct = dv.empty(m)
        self.state = t.zeros(STATE_BYTES, dtype=t.uint8, device=dv.device())
        self.state_host = t.empty(STATE_BYTES, dtype=t.uint8, pin_memory=True)
        self.dy = None
        self.launches = 0
        # (start, end) CUDA events around each cascade on the solver's stream
        # when time_cascade is set (bench.py: the dominant kernels' time
        # inside the real step)
        self.time_cascade = False
        self.cascade_events = []
        # One CUDA graph for the whole iteration (scaling, rhs, [Y|x] seed,
        # x0 + cascade, directions, ratio test, update, objectives, state
        # read-back) when the cascade is the one-CTA kernel: no pivot-block
        # flags, so nothing depends on the epoch and the same graph replays
        # every iteration.  c1 is launch-bound (~15 small launches around a
        # 0.3 ms cascade).  PDAS_NO_GRAPH=1 keeps the eager path.
        self._graph = None
        self._graph_launches = 0
        self._graph_ok = (self.graph_iterations and backend == "woodbury"
                          and not os.environ.get("PDAS_NO_GRAPH")
                          and bool(load().pdas_cascade_one_cta(m, n)))

    # -- iterate I/O (host <-> device), the e2e boundary
    def load_iterate(self, x, y, s) -> None:
        for dst, src in ((self.x, x), (self.y, y), (self.s, s)):
            src = src if not isinstance(src, np.ndarray) else self.t.from_numpy(
                np.ascontiguousarray(src, dtype=np.float64))
            dst.copy_(src, non_blocking=True)

    def read_iterate(self):
        return dv.download(self.x), dv.download(self.y), dv.download(self.s)

    # -- state block helpers
    def _sptr(self, off=0) -> int:
        return dv.ptr(self.state) + off

    def _fetch_state(self) -> PdasIterState:
        self.state_host.copy_(self.state, non_blocking=True)
        dv.synchronize()
        return PdasIterState.from_buffer_copy(self.state_host.numpy().tobytes())

    def objectives(self) -> PdasIterState:
        """gap, c'x, b'y at the current iterate (state otherwise reset)."""
        st = dv.stream()
        call("pdas_iter_reset", self._sptr(), st)
        call("pdas_iter_objectives", dv.ptr(self.x), dv.ptr(self.s), dv.ptr(self.prob.c),
             dv.ptr(self.prob.b), dv.ptr(self.y), self.n, self.m, self._sptr(), st)
        return self._fetch_state()

    # -- the iteration
    def _solve_direct_into(self, dy, fail_ptr) -> None:
        """normal.py:101-105 on device: chol(A diag(d) A^T) w = rhs."""
        m, n = self.m, self.n
        G = d_gram(self.prob.A, m, n, self.d)
        L, _ = d_cholesky(G, m, fail_ptr=fail_ptr)
        dy.copy_(self.rhs)
        d_solve_many(L, m, dy, 1)
        self.launches += 6

    def _tail(self, dy) -> None:
        """solver.py:166-189, 257-260: directions, ratio test, update, gap."""
        st = dv.stream()
        m, n, P = self.m, self.n, self.prob
        call("pdas_iter_directions", dv.ptr(P.A), m, n, dv.ptr(dy), dv.ptr(self.d),
             dv.ptr(self.x), dv.ptr(self.s), dv.ptr(self.dx), dv.ptr(self.ds), self.rho,
             self._sptr(), st)
        call("pdas_iter_update", dv.ptr(self.x), dv.ptr(self.y), dv.ptr(self.s),
             dv.ptr(self.dx), dv.ptr(dy), dv.ptr(self.ds), n, m, self._sptr(), st)
        call("pdas_iter_objectives", dv.ptr(self.x), dv.ptr(self.s), dv.ptr(P.c), dv.ptr(P.b),
             dv.ptr(self.y), n, m, self._sptr(), st)
        self.launches += 7

    def _cascade(self) -> None:
        """solve_sweeps on [Y | x] (normal.py:124), fail word into the state."""
        m, n = self.m, self.n
        self.epoch += 1
        call("pdas_solve_sweeps_ws", dv.ptr(self.cols), dv.ptr(self.prob.A), dv.ptr(self.d), m,
             n, dv.ptr(self.casc_ws), self.epoch, self._sptr(OFF_CASCADE_FAIL), dv.stream())
        self.launches += 2 * ((n + 127) // 128)

    def _cascade_x0(self) -> None:
        """x0 = L0^-T L0^-1 rhs (normal.py:123) fused with the cascade: the
        library overlaps the x0 solve with the Y part when it can."""
        m, n = self.m, self.n
        self.epoch += 1
        call("pdas_solve_sweeps_ws_x0", dv.ptr(self.cols), dv.ptr(self.prob.A), dv.ptr(self.d),
             dv.ptr(self.basis.L0), m, n, dv.ptr(self.casc_ws), self.epoch,
             self._sptr(OFF_CASCADE_FAIL), dv.stream())
        # one-CTA cascade: one kernel (x0 inside); else x0 solve (2) + per pivot
        # block: panel, update, and the x lane's update
        nb = int(load().pdas_cascade_solve_blocks(m, n))
        xlane = n % int(load().pdas_cascade_tile_width(m)) == 0
        self.launches += 1 if nb == 0 else 2 + (3 if xlane else 2) * nb

    def enqueue_solve(self) -> None:
        """Scaling, rhs and the normal-equations solve (cascade or direct)."""
        st = dv.stream()
        m, n, P = self.m, self.n, self.prob
        call("pdas_iter_reset", self._sptr(), st)
        call("pdas_iter_scaling", dv.ptr(self.x), dv.ptr(self.s), n, dv.ptr(self.d),
             self._sptr(), st)
        d_mat_vec(P.A, m, n, self.x, self.rhs)
        self.launches += 4
        if self.backend == "woodbury":
            B = self.basis
            self.cols[:m * n].copy_(B.Y, non_blocking=True)  # init_workspace (normal.py:121-123)
            self.xcol.copy_(self.rhs, non_blocking=True)
            if self.time_cascade:
                ev = (self.t.cuda.Event(enable_timing=True), self.t.cuda.Event(enable_timing=True))
                ev[0].record(self.t.cuda.current_stream())
            self._cascade_x0()
            if self.time_cascade:
                ev[1].record(self.t.cuda.current_stream())
                self.cascade_events.append(ev)
            self.dy = self.xcol
        else:
            self._solve_direct_into(self.dy_direct, self._sptr(OFF_CHOL_FAIL))
            self.dy = self.dy_direct

    def _capture(self) -> None:
        t = self.t
        g = t.cuda.CUDAGraph()
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        n0 = self.launches
        try:
            with t.cuda.graph(g, stream=side):
                self.enqueue_solve()
                self._tail(self.dy)
                self.state_host.copy_(self.state, non_blocking=True)
        finally:
            t.cuda.current_stream().wait_stream(side)
            self._graph_launches = self.launches - n0
            self.launches = n0
        self._graph = g

    def _solve_and_fetch(self) -> PdasIterState:
        if self._graph_ok and not self.time_cascade and self._graph is None:
            try:
                self._capture()
            except RuntimeError:  # capture refused (driver/runtime): eager launches
                self._graph_ok = False
                self.t.cuda.synchronize()
        if self._graph_ok and not self.time_cascade:
            self._graph.replay()
            self.launches += self._graph_launches
            self.dy = self.xcol
            dv.synchronize()
            return PdasIterState.from_buffer_copy(self.state_host.numpy().tobytes())
        self.enqueue_solve()
        self._tail(self.dy)
        return self._fetch_state()

    def iterate(self) -> IterResult:
        """One PDAS iteration on device; returns the host copy of its state."""
        t0 = time.perf_counter()
        st = self._solve_and_fetch()
        if self.backend == "woodbury" and st.cascade_fail != 0 and not not_interior(
                st.interior_flags):
            # SingularUpdate -> retry with the direct solve, flagged (solver.py:161-165)
            self.state[OFF_CASCADE_FAIL:OFF_CASCADE_FAIL + 4].zero_()
            self._solve_direct_into(self.dy_direct, self._sptr(OFF_CHOL_FAIL))
            fb = PdasIterState.fallback.offset
            self.state[fb:fb + 4].copy_(self.t.tensor([1, 0, 0, 0], dtype=self.t.uint8),
                                        non_blocking=True)
            self.dy = self.dy_direct
            self._tail(self.dy)
            st = self._fetch_state()
        return IterResult(st, (time.perf_counter() - t0) * 1e3)

"""Column-sharded Egidi-Maponi cascade: one process per GPU.

Why it shards (reference parallel.py:1-7, _kernels.pyx:260-289, SURVEY.md
§8(e)): inside step l every column k > l of [Y | x] is updated independently;
the only cross-column input is the pivot column l (final after step l-1) and
its denominator.  So columns can live on different GPUs as long as each
finished pivot column reaches every GPU before that GPU applies it.

Ownership (block-cyclic, aligned with the kernels' tiles):
  * pivot block b = pivots [bB, min(bB+B, n)), B = pdas_cascade_block_pivots()
    (128), owned by rank b mod G;
  * column tile t = columns [tw, tw+w) of [Y | x], w = pdas_cascade_tile_width(m),
    owned by the owner of the block its first column falls in (B is a multiple
    of w, so a block's tiles are exactly its columns; the x column n belongs to
    block n div B).
Every rank holds the whole [Y | x] buffer -- Y and x0 are computed redundantly
(deterministic, no exchange) -- but advances only the tiles it owns.

Schedule of one cascade on every rank (`cascade_schedule`):
    panel(0) on owner(0); broadcast block 0
    for b = 0 .. nb-1:
        main stream waits for block b
        side stream: panel(b+1) on owner(b+1) (after its own update(b-1));
                     broadcast block b+1                       (lookahead)
        main stream: update(b) = block b applied to this rank's tiles past
                     block b+1 (past block b at the end)
    broadcast the x column from its owner (unless the last panel covered it)
A block broadcast carries the block's final columns, its denominators and the
fail word, so a breakdown found by the owner of its block stops every rank and
all ranks return the same 1-based step.

Parity: each column receives the pivots in ascending order with the same
per-column arithmetic (tree dot, IEEE divide, unfused multiply-subtract), so
the sharded result is bitwise the 1-GPU cascade (and the reference's) for any
G, B and w (tests/test_dist.py on CPU with gloo, tests/test_gpu_dist.py with
the CUDA blocks).

The schedule is a generator that yields at every collective; the driver
performs it.  `run_collective` does it with torch.distributed (NCCL on GPUs,
gloo in the CPU tests); `run_lockstep` drives G in-process virtual ranks in
lock-step (the broadcast becomes a copy), which is how one GPU checks the
sharded path without running ranks that wait on each other.

Fused exchange (exchange="peer"; EXPERIMENTAL until it has run
on two real GPUs -- so far only virtual ranks on one device and a 1-rank
group have exercised it): instead of broadcasting a
block after its panel, the owner's panel kernel stores each finished tile
from registers straight into every peer's [Y | x] (and denominators, fail
word) through NVLink peer mappings and releases a per-tile flag there
(pdas_cascade_panel_peers); a non-owner's side stream runs a wait kernel on
those flags (pdas_cascade_peer_wait) where it would have joined the
broadcast.  The peer addresses come from torch symmetric memory (one
process per GPU) or, for the in-process virtual ranks, are the other ranks'
buffers on the same device.
"""

from __future__ import annotations

import bisect
import contextlib
from typing import Iterator, List, Optional, Sequence, Tuple

import numpy as np

from .engine import DeviceSolver

Op = Tuple  # ("block", b, src, c0, c1, p0, p1) | ("x", src)


class ShardPlan:
    """Block-cyclic ownership of pivots and column tiles for one rank."""

    def __init__(self, m: int, n: int, world: int, rank: int, block: int, tile: int):
        if world < 1 or not 0 <= rank < world:
            raise ValueError("bad world/rank")
        if tile < 1 or block < tile or block % tile:
            raise ValueError("block must be a positive multiple of the tile width")
        if n < 1:
            raise ValueError("n must be >= 1")
        self.m, self.n, self.world, self.rank = int(m), int(n), int(world), int(rank)
        self.B, self.w = int(block), int(tile)
        self.nb = (self.n + self.B - 1) // self.B
        self.ntiles = (self.n + 1 + self.w - 1) // self.w
        self.tiles = np.array([t for t in range(self.ntiles) if self.tile_owner(t) == rank],
                              dtype=np.int64)
        self._tl = self.tiles.tolist()
        # the last panel's tiles cover column n unless n falls on a tile edge
        self.x_in_last_panel = self.n % self.w != 0
        self.x_owner = self.tile_owner(self.n // self.w)

    def block_owner(self, b: int) -> int:
        return b % self.world

    def tile_owner(self, t: int) -> int:
        return ((t * self.w) // self.B) % self.world

    def owns_block(self, b: int) -> bool:
        return self.block_owner(b) == self.rank

    def block(self, b: int) -> Tuple[int, int]:
        p0 = b * self.B
        return p0, min(p0 + self.B, self.n)

    def panel_bounds(self, b: int) -> Tuple[int, int, int]:
        """(q0, p0, p1): block b after the previous block [q0, p0)."""
        p0, p1 = self.block(b)
        return (p0 - self.B if b > 0 else 0), p0, p1

    def block_columns(self, b: int) -> Tuple[int, int]:
        """Columns a panel over block b finalises (its tiles, clipped at n+1)."""
        p0, p1 = self.block(b)
        return p0, min((p1 + self.w - 1) // self.w * self.w, self.n + 1)

    def update_start(self, b: int) -> int:
        """Index into `tiles` of the first tile update(b) touches."""
        last = self.block(b + 1)[1] if b + 1 < self.nb else self.block(b)[1]
        t0 = (last + self.w - 1) // self.w
        return bisect.bisect_left(self._tl, t0)

    def update_start_chained(self, b: int) -> int:
        """Chained schedule: update(b) also covers block b+1's tiles (the early
        panel of block b+1 waits for them on its own rank)."""
        if b + 1 < self.nb:
            t0 = self.block(b + 1)[0] // self.w
        else:
            t0 = (self.block(b)[1] + self.w - 1) // self.w
        return bisect.bisect_left(self._tl, t0)

    def block_op(self, b: int) -> Op:
        c0, c1 = self.block_columns(b)
        p0, p1 = self.block(b)
        return ("block", b, self.block_owner(b), c0, c1, p0, p1)


class _NullBackend:
    """Stream hooks are no-ops unless a backend overrides them."""

    def begin(self) -> None:
        pass

    def side(self):
        return contextlib.nullcontext()

    def main_wait_side(self) -> None:
        pass

    def side_wait_update(self) -> None:
        pass

    def mark_update(self) -> None:
        pass

    def block_final(self, b: int) -> None:
        pass

    def mark_before_update(self) -> None:
        pass

    def end(self) -> None:
        pass


def cascade_schedule(plan: ShardPlan, be) -> Iterator[Op]:
    """One sharded cascade on this rank; yields each collective (see module doc).

    `be` provides panel(q0, p0, p1, tag), update(p0, p1, i0, tag) (tiles
    plan.tiles[i0:]) and the stream hooks of _NullBackend.

    be.chained (the 1-GPU engine's early-panel order, r02): update(b) on the
    owner of block b+1 covers block b+1's tiles first and tags them b+1; the
    panel of block b+1 then applies no previous block itself (q0 = p0) and
    waits in-kernel for those tags -- 2B instead of 3B dependent steps per
    block on the serial chain, the multi-GPU ceiling."""
    if getattr(be, "chained", False):
        yield from _chained_schedule(plan, be)
        return
    be.begin()
    with be.side():
        if plan.owns_block(0):
            be.panel(*plan.panel_bounds(0))
        yield plan.block_op(0)
    for b in range(plan.nb):
        be.main_wait_side()  # block b is final here
        be.block_final(b)
        if b + 1 < plan.nb:
            with be.side():
                if plan.owns_block(b + 1):
                    be.side_wait_update()  # this rank's update(b-1) reached block b+1
                    be.panel(*plan.panel_bounds(b + 1))
                yield plan.block_op(b + 1)
        i0 = plan.update_start(b)
        if i0 < len(plan.tiles):
            be.update(*plan.block(b), i0)
        be.mark_update()
    be.main_wait_side()
    be.end()
    if not plan.x_in_last_panel:
        yield ("x", plan.x_owner)


def _chained_schedule(plan: ShardPlan, be) -> Iterator[Op]:
    be.begin()
    with be.side():
        if plan.owns_block(0):
            p0, p1 = plan.block(0)
            be.panel(p0, p0, p1, tag=0)
        yield plan.block_op(0)
    for b in range(plan.nb):
        be.main_wait_side()  # block b is final here
        be.block_final(b)
        be.mark_before_update()  # the main stream up to update(b-1)
        i0 = plan.update_start_chained(b)
        if i0 < len(plan.tiles):
            be.update(*plan.block(b), i0, tag=b + 1)
        be.mark_update()
        if b + 1 < plan.nb:
            with be.side():
                if plan.owns_block(b + 1):
                    # not resident while update(b-1) still runs; waits in-kernel
                    # for this rank's update(b) of its own tiles
                    be.side_wait_update()
                    p0, p1 = plan.block(b + 1)
                    be.panel(p0, p0, p1, tag=b + 1)
                yield plan.block_op(b + 1)
    be.main_wait_side()
    be.end()
    if not plan.x_in_last_panel:
        yield ("x", plan.x_owner)


# ------------------------------------------------------------------ drivers
def run_collective(plan: ShardPlan, be, group=None) -> None:
    """Drive the schedule with torch.distributed broadcasts over `group`.

    `be.block_views(c0, c1, p0, p1)` returns the tensors a block broadcast
    carries (columns, denominators, fail word); `be.x_view()` the x column.
    Each broadcast is issued under the stream the schedule is on.  A backend
    with `fused` set exchanges blocks itself (`be.exchange_block(op)`: the
    owner's panel already stored them into the peers; others wait)."""
    import torch.distributed as dist

    ranks = None if group is None else dist.get_process_group_ranks(group)

    def g(src):
        return src if ranks is None else ranks[src]

    fused = getattr(be, "fused", False)
    for op in cascade_schedule(plan, be):
        if op[0] == "block" and fused:
            be.exchange_block(op)
        elif op[0] == "block":
            _, b, src, c0, c1, p0, p1 = op
            views = be.block_views(c0, c1, p0, p1)
            pack = getattr(be, "pack_scalars", None)
            if pack is not None:
                # one payload for the block's columns, one for its denominators
                # and the fail word (packed by the owner, unpacked by the rest)
                dist.broadcast(views[0], g(src), group=group)
                small = pack(p0, p1, src == plan.rank)
                dist.broadcast(small, g(src), group=group)
                be.unpack_scalars(p0, p1, small, src == plan.rank)
            else:
                for t in views:
                    dist.broadcast(t, g(src), group=group)
        else:
            dist.broadcast(be.x_view(), g(op[1]), group=group)


def run_lockstep(plans: Sequence[ShardPlan], bes: Sequence) -> None:
    """Drive G virtual ranks in one process: every rank advances to its next
    collective, then the owner's views are copied into the others'."""
    gens = [cascade_schedule(p, be) for p, be in zip(plans, bes)]
    while True:
        ops = [next(gn, None) for gn in gens]
        if all(o is None for o in ops):
            return
        if any(o != ops[0] for o in ops):
            raise RuntimeError(f"virtual ranks diverged: {ops}")
        op = ops[0]
        if op[0] == "block" and all(getattr(be, "fused", False) for be in bes):
            for be in bes:
                be.exchange_block(op)
        elif op[0] == "block":
            _, b, src, c0, c1, p0, p1 = op
            srcv = bes[src].block_views(c0, c1, p0, p1)
            for r, be in enumerate(bes):
                if r != src:
                    for dst, s in zip(be.block_views(c0, c1, p0, p1), srcv):
                        dst.copy_(s)
        else:
            src = op[1]
            for r, be in enumerate(bes):
                if r != src:
                    be.x_view().copy_(bes[src].x_view())


# ------------------------------------------------------------------ CUDA backend
class CudaShard(_NullBackend):
    """The CUDA building blocks (pdas_cascade_panel / pdas_cascade_update) on
    one rank's buffers.  cols: flat m*(n+1) fp64; a: flat m*n; d: n; ws: the
    pdas_cascade_ws_bytes workspace (zeroed once); fail: 4-byte device view.

    streams=True: panels + block broadcasts on a high-priority side stream,
    updates on the caller's stream (the lookahead of the 1-GPU cascade)."""

    def __init__(self, plan: ShardPlan, cols, a, d, ws, fail, streams: bool = True,
                 peers: Optional[Sequence[Tuple[int, int, int]]] = None, x0_low=None):
        """peers: for the fused exchange, (cols, ws, fail) device addresses of
        every OTHER rank, in rank order, valid in this process; None = the
        blocks travel by broadcast (run_collective) or copy (run_lockstep).
        x0_low: L0 -- the x0 = L0^-T L0^-1 rhs solve (normal.py:123) joins the
        cascade: on the x column's owner it runs on its own stream (the x
        lane) together with that tile's per-block updates, off the critical
        path, when column n sits alone in its tile; other ranks skip it (they
        receive x at the end).  Without an x lane the owner solves first."""
        import ctypes

        from . import _device as dv
        from ._lib import call

        t = dv.require_gpu()
        self.t, self.dv, self.call = t, dv, call
        self.plan = plan
        self.cols, self.a, self.d, self.ws, self.fail = cols, a, d, ws, fail
        nd = max(plan.n, 1)
        self.denoms = ws[: nd * 8].view(t.float64)
        self.tiles = t.from_numpy(plan.tiles.copy()).to(dv.device())
        self.epoch = 0
        self.streams = streams
        self.fused = peers is not None
        if self.fused:
            if len(peers) != plan.world - 1:
                raise ValueError("peers must list every other rank")
            arr = ctypes.c_uint64 * max(len(peers), 1)
            self._peer_arrays = tuple(arr(*[int(p[i]) for p in peers]) for i in range(3))
        if streams:
            lo, hi = t.cuda.Stream.priority_range()
            self.side_stream = t.cuda.Stream(priority=hi)
            self.ev_update = t.cuda.Event()
        self.main = None
        # the chained (early-panel) schedule for the broadcast exchange; the
        # experimental fused peer exchange keeps the previous-block panels
        self.chained = not self.fused
        self.x0_low = x0_low
        x_tile = plan.n // plan.w
        self.xlane = (x0_low is not None and streams and not plan.x_in_last_panel
                      and plan.rank == plan.x_owner)
        if self.xlane:
            # the x tile leaves the owner's regular update list
            keep = plan.tiles[plan.tiles != x_tile]
            self.tiles = t.from_numpy(keep.copy()).to(dv.device())
            self._ntiles = len(keep)
            start = plan.update_start_chained if self.chained else plan.update_start
            self._starts = [int(np.searchsorted(keep, plan.tiles[start(b)])
                                if start(b) < len(plan.tiles) else len(keep))
                            for b in range(plan.nb)]
            self.x_tiles = t.tensor([x_tile], dtype=t.int64, device=dv.device())
            self.x_stream = t.cuda.Stream(priority=hi)
            self.ev_block = t.cuda.Event()
            self.x_work = t.empty(int(plan.m), dtype=t.float64, device=dv.device())
        else:
            self._ntiles = len(plan.tiles)
            self._starts = None
        self._scal = t.empty(plan.B + 1, dtype=t.float64, device=dv.device())

    def reset(self, cols, d):
        self.cols, self.d = cols, d

    # -- stream hooks
    def begin(self) -> None:
        self.epoch += 1
        if not self.fused:  # fused: the caller zeroes it before the peers may write it
            self.fail.zero_()
        if self.chained:
            self.call("pdas_cascade_reset_tags", self.dv.ptr(self.ws), self.plan.n,
                      self.dv.stream())
        if self.streams:
            self.main = self.t.cuda.current_stream()
            self.side_stream.wait_stream(self.main)
            self.ev_update.record(self.main)
        if self.x0_low is not None:
            m, n = self.plan.m, self.plan.n
            xcol = self.cols[n * m:(n + 1) * m]
            if self.xlane:
                self.x_stream.wait_stream(self.main)
                with self.t.cuda.stream(self.x_stream):
                    self.call("pdas_cholesky_solve_one", self.dv.ptr(self.x0_low), m,
                              self.dv.ptr(xcol), self.dv.stream())
            elif self.plan.rank == self.plan.x_owner:
                self.call("pdas_cholesky_solve_one", self.dv.ptr(self.x0_low), m,
                          self.dv.ptr(xcol), self.dv.stream())

    def block_final(self, b: int) -> None:
        """x lane: block b is final on the main stream -> the x tile gets it."""
        if not self.xlane:
            return
        p = self.plan
        p0, p1 = p.block(b)
        self.ev_block.record(self.main)
        self.x_stream.wait_event(self.ev_block)
        with self.t.cuda.stream(self.x_stream):
            self.call("pdas_cascade_update", self.dv.ptr(self.cols), self.dv.ptr(self.a),
                      self.dv.ptr(self.d), p.m, p.n, p0, p1, self.dv.ptr(self.x_tiles), 1,
                      self.dv.ptr(self.ws), self.dv.ptr(self.fail), self.dv.stream())

    def end(self) -> None:
        if self.xlane:
            self.main.wait_stream(self.x_stream)

    def side(self):
        return self.t.cuda.stream(self.side_stream) if self.streams else contextlib.nullcontext()

    def main_wait_side(self) -> None:
        if self.streams:
            self.main.wait_stream(self.side_stream)

    def side_wait_update(self) -> None:
        if self.streams:
            self.side_stream.wait_event(self.ev_update)

    def mark_update(self) -> None:
        if self.streams and not self.chained:
            self.ev_update.record(self.main)

    def mark_before_update(self) -> None:
        if self.streams:
            self.ev_update.record(self.main)

    # -- compute
    def panel(self, q0: int, p0: int, p1: int, tag: int = 0) -> None:
        p, dv = self.plan, self.dv
        if self.chained:
            self.call("pdas_cascade_panel_chained", dv.ptr(self.cols), dv.ptr(self.a),
                      dv.ptr(self.d), p.m, p.n, p0, p1, dv.ptr(self.ws), self.epoch,
                      dv.ptr(self.fail), tag, dv.stream())
            return
        if self.fused:
            pc, pw, pf = self._peer_arrays
            self.call("pdas_cascade_panel_peers", dv.ptr(self.cols), dv.ptr(self.a),
                      dv.ptr(self.d), p.m, p.n, q0, p0, p1, dv.ptr(self.ws), self.epoch,
                      dv.ptr(self.fail), p.world - 1, pc, pw, pf, dv.stream())
            return
        self.call("pdas_cascade_panel", dv.ptr(self.cols), dv.ptr(self.a), dv.ptr(self.d), p.m,
                  p.n, q0, p0, p1, dv.ptr(self.ws), self.epoch, dv.ptr(self.fail), dv.stream())

    def exchange_block(self, op: Op) -> None:
        """Fused exchange of a block: nothing to do on its owner (the panel
        stored it into the peers); elsewhere the current stream waits for the
        owner's per-tile flags."""
        _, b, src, c0, c1, p0, p1 = op
        if src == self.plan.rank:
            return
        p, dv = self.plan, self.dv
        self.call("pdas_cascade_peer_wait", dv.ptr(self.ws), p.m, p.n, c0, c1, self.epoch,
                  dv.stream())

    def update(self, p0: int, p1: int, i0: int, tag: int = 0) -> None:
        p, dv = self.plan, self.dv
        if self._starts is not None:  # x lane: index into the list without the x tile
            i0 = self._starts[p0 // p.B]
        if i0 >= self._ntiles:
            return
        if tag > 0:
            self.call("pdas_cascade_update_tagged", dv.ptr(self.cols), dv.ptr(self.a),
                      dv.ptr(self.d), p.m, p.n, p0, p1, dv.ptr(self.tiles) + 8 * i0,
                      self._ntiles - i0, dv.ptr(self.ws), dv.ptr(self.fail), tag, dv.stream())
            return
        self.call("pdas_cascade_update", dv.ptr(self.cols), dv.ptr(self.a), dv.ptr(self.d), p.m,
                  p.n, p0, p1, dv.ptr(self.tiles) + 8 * i0, self._ntiles - i0, dv.ptr(self.ws),
                  dv.ptr(self.fail), dv.stream())

    def pack_scalars(self, p0: int, p1: int, owner: bool):
        """[denominators of block [p0, p1) | fail word] as one payload."""
        sc = self._scal[: p1 - p0 + 1]
        if owner:
            sc[: p1 - p0].copy_(self.denoms[p0:p1])
            sc[p1 - p0:].copy_(self._fail32().to(self.t.float64))
        return sc

    def _fail32(self):
        # the fail word is an int32, possibly viewed as 4 bytes of the state block
        return self.fail.view(self.t.int32) if self.fail.dtype == self.t.uint8 else self.fail

    def unpack_scalars(self, p0: int, p1: int, sc, owner: bool) -> None:
        if owner:
            return
        self.denoms[p0:p1].copy_(sc[: p1 - p0])
        self._fail32().copy_(sc[p1 - p0:].to(self.t.int32))

    # -- collective payloads
    def block_views(self, c0, c1, p0, p1):
        m = self.plan.m
        return [self.cols[c0 * m:c1 * m], self.denoms[p0:p1], self.fail]

    def x_view(self):
        m, n = self.plan.m, self.plan.n
        return self.cols[n * m:(n + 1) * m]


def cascade_tile_width(m: int) -> int:
    from ._lib import load

    w = int(load().pdas_cascade_tile_width(m))
    if w < 1:
        raise ValueError(f"no cascade configuration for m={m}")
    return w


def cascade_block_pivots() -> int:
    from ._lib import load

    return int(load().pdas_cascade_block_pivots())


def make_plan(m: int, n: int, world: int, rank: int, block: Optional[int] = None) -> ShardPlan:
    w = cascade_tile_width(m)
    B = block or cascade_block_pivots()
    return ShardPlan(m, n, world, rank, B, w)


class ShardedSolver(DeviceSolver):
    """DeviceSolver whose cascade runs column-sharded over a process group
    (one process per GPU, NCCL).  Everything else of the iteration -- scaling,
    A x, x0, A^T dy, ratio test, update -- is replicated on every rank (same
    kernels, same bits), so the only traffic is the cascade's block
    broadcasts plus one x-column broadcast per iteration."""

    graph_iterations = False  # collectives and the per-rank schedule: eager

    def __init__(self, prob, group=None, rho: float = 0.9, basis=None, L0=None,
                 block: Optional[int] = None, exchange: str = "nccl"):
        """exchange: "nccl" (a broadcast per block) or "peer" (the fused
        exchange: [Y | x], the cascade workspace and the fail word live in
        torch symmetric memory and the owner's panel stores into the peers)."""
        import torch.distributed as dist

        from ._lib import OFF_CASCADE_FAIL

        if exchange not in ("nccl", "peer"):
            raise ValueError(f"exchange must be 'nccl' or 'peer', not {exchange!r}")
        super().__init__(prob, "woodbury", rho, basis=basis, L0=L0)
        self.group = group
        self.exchange = exchange
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self.plan = make_plan(self.m, self.n, world, rank, block)
        self._state_fail = self.state[OFF_CASCADE_FAIL:OFF_CASCADE_FAIL + 4]
        peers = None
        fail = self._state_fail
        if exchange == "peer":
            fail, peers = self._symmetric_buffers(world, rank)
        self.shard = CudaShard(self.plan, self.cols, prob.A, self.d, self.casc_ws, fail,
                               peers=peers, x0_low=self.basis.L0)
        p = self.plan
        self._casc_launches = sum(1 for b in range(p.nb) if p.owns_block(b)) + sum(
            1 for b in range(p.nb) if p.update_start(b) < len(p.tiles))

    def _symmetric_buffers(self, world: int, rank: int):
        """Move [Y | x], the cascade workspace and a fail word into one
        symmetric-memory allocation; return (fail view, peer addresses)."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        t, m, n = self.t, self.m, self.n
        from . import _device as dv

        def up(x):
            return (x + 255) // 256 * 256

        ncol = m * (n + 1) * 8
        wsb = self.casc_ws.numel()
        off_ws = up(ncol)
        off_fail = up(off_ws + wsb)
        buf = symm.empty(off_fail + 256, dtype=t.uint8, device=dv.device())
        buf.zero_()
        g = self.group if self.group is not None else dist.group.WORLD
        handle = symm.rendezvous(buf, g.group_name)
        ptrs = [int(p) for p in handle.buffer_ptrs]
        self._symm = (buf, handle)
        self.cols = buf[:ncol].view(t.float64)
        self.xcol = self.cols[m * n:]
        self.casc_ws = buf[off_ws:off_ws + wsb]
        fail = buf[off_fail:off_fail + 4].view(t.int32)
        self._sync = t.zeros(1, dtype=t.int32, device=dv.device())
        peers = [(ptrs[r], ptrs[r] + off_ws, ptrs[r] + off_fail) for r in range(world)
                 if r != rank]
        return fail, peers

    def _cascade(self) -> None:
        if self.exchange == "peer":
            import torch.distributed as dist

            # every rank has re-seeded [Y | x] and finished the previous
            # cascade before any peer's panel may store into it
            self.shard.fail.zero_()
            dist.all_reduce(self._sync, group=self.group)
            run_collective(self.plan, self.shard, self.group)
            self._state_fail.copy_(self.shard.fail.view(self.t.uint8))
        else:
            run_collective(self.plan, self.shard, self.group)
        self.launches += self._casc_launches

    def _cascade_x0(self) -> None:
        # x0 (normal.py:123) is solved inside the schedule: on the x column's
        # owner, on the x lane, overlapped with the cascade (CudaShard.begin)
        self.launches += 2 if self.plan.rank == self.plan.x_owner else 0
        self._cascade()


def solve_sweeps_virtual(cols: np.ndarray, a: np.ndarray, d: np.ndarray, world: int,
                         block: Optional[int] = None, fused: bool = False,
                         reps: int = 1) -> Tuple[int, List[np.ndarray]]:
    """The sharded cascade over `world` virtual ranks on the current GPU, in
    lock-step (no rank waits on another inside a kernel).  Returns the common
    fail code and every rank's final [Y | x] (host copies, column-major).
    fused: blocks move by the panel's peer stores + flag waits (the other
    virtual ranks' buffers stand in for the NVLink peer mappings); by the
    time a rank's wait kernel runs, the owner's panel has been enqueued
    before it on the same stream.  reps > 1 re-runs the cascade from the same
    input (new epoch each time: stale flags of the previous run must not
    satisfy a wait).  Verification entry point for the multi-GPU schedule."""
    from . import _device as dv
    from ._lib import load

    t = dv.require_gpu()
    m, n = a.shape
    A = dv.upload(np.asfortranarray(a))
    dd = dv.upload(np.ascontiguousarray(d, dtype=np.float64))
    wsb = int(load().pdas_cascade_ws_bytes(m, n))
    plans, bufs, bes = [], [], []
    c_in = dv.upload(np.asfortranarray(cols))
    for r in range(world):
        plans.append(make_plan(m, n, world, r, block))
        bufs.append((c_in.clone(), t.zeros(wsb, dtype=t.uint8, device=dv.device()),
                     t.zeros(1, dtype=t.int32, device=dv.device())))
    for r in range(world):
        peers = None
        if fused:
            peers = [tuple(dv.ptr(x) for x in bufs[q]) for q in range(world) if q != r]
        c, ws, fail = bufs[r]
        bes.append(CudaShard(plans[r], c, A, dd, ws, fail, streams=False, peers=peers))
    for rep in range(reps):
        for (c, _, fail) in bufs:
            c.copy_(c_in)
            fail.zero_()
        run_lockstep(plans, bes)
    dv.synchronize()
    fails = [int(be.fail.item()) for be in bes]
    if len(set(fails)) != 1:
        raise RuntimeError(f"ranks disagree on the breakdown step: {fails}")
    outs = [dv.download(be.cols).reshape((m, n + 1), order="F") for be in bes]
    return fails[0], outs

"""Sharded cascade schedule (paper_1502_03543_b200/dist.py) on CPU.

The schedule and ownership logic are driven with an oracle backend: the
panel / update building blocks restated with the oracle's sweep phases
(oracle/pdas_oracle.c, _kernels.pyx:205-231), broadcasts over torch.distributed
gloo (world_size 2 and 3, real processes) or the in-process lock-step driver.
Every rank's final [Y | x] must be bitwise the serial cascade
(or_solve_sweeps, _kernels.pyx:234-291) and every rank must return the same
breakdown step."""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import bits_equal
from oracle import oracle as O
from paper_1502_03543_b200 import dist as D


class OracleShard(D._NullBackend):
    """panel/update of one rank, restated on the CPU with the oracle."""

    def __init__(self, plan, cols, a, d):
        self.K = O.restated()
        self.plan = plan
        m, n = a.shape
        self.flat = np.array(np.asfortranarray(cols).ravel(order="F"), copy=True)
        self.cols = self.flat.reshape((m, n + 1), order="F")
        self.a = np.asfortranarray(a)
        self.d = np.ascontiguousarray(d, dtype=np.float64)
        self.denoms = np.zeros(max(n, 1))
        self.fail = np.zeros(1, dtype=np.int32)
        self.inner = np.zeros(n + 1)
        self.v = np.zeros(m)

    def _apply(self, l, k0, k1):
        if self.d[l] == 1.0 or k0 >= k1:
            return
        self.K.build_v(self.a, l, self.d[l], self.v)
        self.K.sweep_phase1(self.cols, self.v, self.inner, k0, k1)
        self.K.sweep_phase2(self.cols, l, self.inner, self.denoms[l], k0, k1)

    def panel(self, q0, p0, p1):
        if self.fail[0]:
            return
        e = min((p1 + self.plan.w - 1) // self.plan.w * self.plan.w, self.plan.n + 1)
        for l in range(q0, p0):
            self._apply(l, p0, e)
        for l in range(p0, p1):
            if self.d[l] == 1.0:
                continue
            self.K.build_v(self.a, l, self.d[l], self.v)
            self.K.sweep_phase1(self.cols, self.v, self.inner, l, e)
            den = 1.0 + self.inner[l]
            if abs(den) <= O.RestatedKernels.DENOM_EPS_REL * (1.0 + abs(self.inner[l])):
                self.fail[0] = l + 1
                return
            self.denoms[l] = den
            self.K.sweep_phase2(self.cols, l, self.inner, den, l + 1, e)

    def update(self, p0, p1, i0):
        if self.fail[0]:
            return
        w, n = self.plan.w, self.plan.n
        ranges = []
        for t in self.plan.tiles[i0:]:
            c0, c1 = int(t) * w, min(int(t) * w + w, n + 1)
            if ranges and ranges[-1][1] == c0:
                ranges[-1][1] = c1
            else:
                ranges.append([c0, c1])
        for l in range(p0, p1):
            for c0, c1 in ranges:
                self._apply(l, c0, c1)

    def block_views(self, c0, c1, p0, p1):
        m = self.plan.m
        return [torch.from_numpy(self.flat[c0 * m:c1 * m]), torch.from_numpy(self.denoms[p0:p1]),
                torch.from_numpy(self.fail)]

    def x_view(self):
        m, n = self.plan.m, self.plan.n
        return torch.from_numpy(self.flat[n * m:(n + 1) * m])


def _system(m, n, seed, skip=0.15, spread=3.0):
    rng = np.random.default_rng(seed)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = np.power(10.0, rng.uniform(-spread, spread, n))
    d[rng.random(n) < skip] = 1.0
    cols = np.asfortranarray(rng.uniform(-1, 1, (m, n + 1)))
    return a, d, cols


def _serial(a, d, cols):
    m, n = a.shape
    c = cols.copy(order="F")
    ret = O.restated().solve_sweeps(c, a, d, np.zeros(n + 1), np.zeros(m), 1)
    return ret, c


def _breakdown_d(a, d, cols, step):
    """d with a breakdown exactly at pivot `step` (0-based): d_l = 1 - 1/q,
    q = a_l . col_l after the serial steps < l (so 1 + inner_l rounds to ~0)."""
    m, n = a.shape
    K = O.restated()
    c = cols.copy(order="F")
    assert K.solve_sweeps_prefix(c, a, d, np.zeros(n + 1), np.zeros(m), step, 1) == 0
    q = K.dot_tree(a[:, step], c[:, step])
    d2 = d.copy()
    d2[step] = 1.0 - 1.0 / q
    return d2


class ChainedOracleShard(OracleShard):
    """The chained (early-panel) schedule: update(b) covers block b+1's tiles,
    the panel applies no previous block (the GPU form waits on tile tags)."""

    chained = True

    def panel(self, q0, p0, p1, tag=0):
        assert q0 == p0
        super().panel(q0, p0, p1)

    def update(self, p0, p1, i0, tag=0):
        super().update(p0, p1, i0)


def _lockstep(a, d, cols, world, B, w, chained=False):
    m, n = a.shape
    plans = [D.ShardPlan(m, n, world, r, B, w) for r in range(world)]
    cls = ChainedOracleShard if chained else OracleShard
    bes = [cls(p, cols, a, d) for p in plans]
    D.run_lockstep(plans, bes)
    return [int(be.fail[0]) for be in bes], [be.cols for be in bes]


def test_plan_ownership():
    p = D.ShardPlan(10, 100, 3, 1, 8, 4)
    assert p.nb == 13 and p.ntiles == 26
    assert all(p.tile_owner(t) == 1 for t in p.tiles)
    assert sorted(sum((D.ShardPlan(10, 100, 3, r, 8, 4).tiles.tolist() for r in range(3)),
                      [])) == list(range(26))
    assert not p.x_in_last_panel and p.x_owner == (100 // 8) % 3
    assert p.panel_bounds(0) == (0, 0, 8) and p.panel_bounds(5) == (32, 40, 48)
    assert p.block_columns(12) == (96, 100)
    q = D.ShardPlan(10, 101, 2, 0, 8, 4)
    assert q.x_in_last_panel and q.block_columns(12) == (96, 102)
    with pytest.raises(ValueError):
        D.ShardPlan(10, 100, 2, 0, 6, 4)


@pytest.mark.parametrize("m,n,world,B,w", [
    (5, 1, 2, 2, 1), (5, 7, 2, 2, 1), (7, 45, 2, 4, 2), (7, 40, 2, 8, 4), (9, 41, 3, 8, 4),
    (6, 64, 4, 16, 8), (12, 63, 5, 8, 8), (3, 30, 1, 4, 2), (16, 100, 3, 16, 16),
])
@pytest.mark.parametrize("chained", [False, True])
def test_lockstep_bitwise(m, n, world, B, w, chained):
    a, d, cols = _system(m, n, 31 * m + n)
    ret, ref = _serial(a, d, cols)
    assert ret == 0
    fails, outs = _lockstep(a, d, cols, world, B, w, chained)
    assert fails == [0] * world
    for c in outs:
        assert bits_equal(c, ref)


@pytest.mark.parametrize("step", [0, 5, 13, 38])
def test_lockstep_breakdown(step):
    m, n = 6, 41
    a, d, cols = _system(m, n, 7, skip=0.0)
    d = _breakdown_d(a, d, cols, step)
    ret, _ = _serial(a, d, cols)
    assert ret == step + 1
    fails, _ = _lockstep(a, d, cols, 3, 4, 2)
    assert fails == [step + 1] * 3
    fails, _ = _lockstep(a, d, cols, 3, 4, 2, chained=True)
    assert fails == [step + 1] * 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, chained=False):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for (m, n, B, w, seed, step) in cases:
            a, d, cols = _system(m, n, seed, skip=0.0 if step is not None else 0.15)
            if step is not None:
                d = _breakdown_d(a, d, cols, step)
            ret, ref = _serial(a, d, cols)
            plan = D.ShardPlan(m, n, world, rank, B, w)
            be = (ChainedOracleShard if chained else OracleShard)(plan, cols, a, d)
            D.run_collective(plan, be)
            assert int(be.fail[0]) == ret, (m, n, rank, int(be.fail[0]), ret)
            if ret == 0:
                assert bits_equal(be.cols, ref), (m, n, B, w, rank)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chained", [(2, False), (3, False), (2, True), (3, True)])
def test_gloo_processes_bitwise(world, chained):
    import torch.multiprocessing as mp

    cases = [(7, 45, 4, 2, 1, None), (8, 40, 8, 4, 2, None), (5, 33, 8, 8, 3, None),
             (6, 41, 4, 2, 7, 22)]
    mp.spawn(_worker, args=(world, _free_port(), cases, chained), nprocs=world, join=True)


class FusedOracleShard(OracleShard):
    """The fused exchange's contract on CPU: the owner's panel itself stores
    the block's final columns, denominators and fail word into every peer and
    raises a per-(epoch, tile) flag there; a non-owner's exchange_block only
    checks that its flags are up (the GPU wait kernel)."""

    fused = True

    def __init__(self, plan, cols, a, d):
        super().__init__(plan, cols, a, d)
        self.peers = []
        self.flags = set()
        self.epoch = 0

    def begin(self):
        self.epoch += 1

    def panel(self, q0, p0, p1):
        super().panel(q0, p0, p1)
        c0, c1 = self.plan.block_columns(p0 // self.plan.B)
        m, w = self.plan.m, self.plan.w
        for peer in self.peers:
            if not self.fail[0]:
                peer.flat[c0 * m:c1 * m] = self.flat[c0 * m:c1 * m]
                peer.denoms[p0:p1] = self.denoms[p0:p1]
            else:
                peer.fail[0] = self.fail[0]
            peer.flags.update((self.epoch, t) for t in range(c0 // w, (c1 + w - 1) // w))

    def exchange_block(self, op):
        _, b, src, c0, c1, p0, p1 = op
        if src != self.plan.rank:
            w = self.plan.w
            missing = [t for t in range(c0 // w, (c1 + w - 1) // w) if (self.epoch, t) not in self.flags]
            assert not missing, (self.plan.rank, b, missing)


@pytest.mark.parametrize("m,n,world,B,w,step", [
    (7, 45, 2, 4, 2, None), (9, 41, 3, 8, 4, None), (6, 64, 4, 16, 8, None),
    (12, 63, 5, 8, 8, None), (6, 41, 3, 4, 2, 22), (6, 41, 3, 4, 2, 0),
])
def test_lockstep_fused_exchange(m, n, world, B, w, step):
    a, d, cols = _system(m, n, 13 * m + n, skip=0.0 if step is not None else 0.15)
    if step is not None:
        d = _breakdown_d(a, d, cols, step)
    ret, ref = _serial(a, d, cols)
    plans = [D.ShardPlan(m, n, world, r, B, w) for r in range(world)]
    bes = [FusedOracleShard(p, cols, a, d) for p in plans]
    for be in bes:
        be.peers = [q for q in bes if q is not be]
    D.run_lockstep(plans, bes)
    assert [int(be.fail[0]) for be in bes] == [ret] * world
    if ret == 0:
        for be in bes:
            assert bits_equal(be.cols, ref)

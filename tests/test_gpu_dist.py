"""The sharded cascade's CUDA building blocks (pdas_cascade_panel /
pdas_cascade_update) under the multi-GPU schedule of dist.py.

One GPU cannot host ranks that wait on one another, so the G-rank schedule
runs as G virtual ranks in lock-step (each with its own [Y | x], workspace
and fail word; a broadcast is a device copy).  Every rank's result must be
bitwise the serial oracle cascade (_kernels.pyx:234-291).  The real
collective driver (NCCL, side-stream lookahead) is exercised with a
one-rank NCCL group through solve_lp(group=...).

The fused exchange (pdas_cascade_panel_peers / pdas_cascade_peer_wait: the
owner's panel stores its tiles into the peers' buffers and flags them) runs
the same way: the virtual ranks' buffers stand in for NVLink peer mappings,
and each wait kernel is enqueued after the owner's panel, so no kernel ever
waits on one that has not been launched."""

import socket

import numpy as np
import pytest

from conftest import bits_equal, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _system(m, n, seed, skip=0.1, spread=3.0):
    rng = np.random.default_rng(seed)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    d = np.power(10.0, rng.uniform(-spread, spread, n))
    d[rng.random(n) < skip] = 1.0
    if m > n or m > 2000:  # no Woodbury basis: a random [Y | x] exercises the same arithmetic
        return a, d, np.asfortranarray(rng.uniform(-1, 1, (m, n + 1)) / np.sqrt(m))
    R = O.restated()
    basis = O.prepare_woodbury(R, a)
    cols, _, _ = O.init_workspace(R, basis, rng.uniform(-1, 1, m))
    return a, d, np.asfortranarray(cols)


def _serial(a, d, cols):
    m, n = a.shape
    c = cols.copy(order="F")
    return O.restated().solve_sweeps(c, a, d, np.zeros(n + 1), np.zeros(m), 8), c


# tile widths 8 / 16 / 8 / 4 / 2 across the register-tile configurations; blocks
# of one tile, two tiles and the default 128; n on and off tile/block edges
@pytest.mark.parametrize("m,n,world,block", [
    (40, 300, 2, None), (40, 256, 3, 8), (64, 129, 2, 16), (200, 700, 3, 16), (300, 520, 2, 32),
    (500, 1000, 4, None), (700, 1200, 3, 64), (1000, 1100, 2, None), (1000, 1024, 5, 16),
    (2000, 2100, 3, None), (2000, 2048, 2, 8), (3000, 300, 2, 4), (5000, 200, 3, 2),
])
def test_virtual_ranks_bitwise(gpu, m, n, world, block):
    from paper_1502_03543_b200 import dist as D

    a, d, cols = _system(m, n, 7 * m + n + world)
    ret, ref = _serial(a, d, cols)
    assert ret == 0
    fail, outs = D.solve_sweeps_virtual(cols, a, d, world, block)
    assert fail == 0
    for r, c in enumerate(outs):
        assert bits_equal(c, ref), r


@pytest.mark.parametrize("m,n,world,block", [
    (40, 300, 2, None), (64, 129, 3, 16), (300, 520, 8, 32), (500, 1000, 4, None),
    (1000, 1024, 5, 16), (2000, 2100, 3, None), (2000, 2048, 8, 8), (3000, 300, 2, 4),
])
def test_virtual_ranks_fused_exchange_bitwise(gpu, m, n, world, block):
    from paper_1502_03543_b200 import dist as D

    a, d, cols = _system(m, n, 5 * m + n + world)
    ret, ref = _serial(a, d, cols)
    assert ret == 0
    # two runs: the second must not be satisfied by the first run's flags
    fail, outs = D.solve_sweeps_virtual(cols, a, d, world, block, fused=True, reps=2)
    assert fail == 0
    for r, c in enumerate(outs):
        assert bits_equal(c, ref), r


@pytest.mark.parametrize("step", [3, 130, 517])
def test_virtual_ranks_fused_breakdown(gpu, step):
    """A breakdown in a block owned by one rank reaches the others through the
    panel's peer fail-word store; every rank returns the same 1-based step."""
    from paper_1502_03543_b200 import dist as D

    m, n = 100, 600
    a, d, cols = _system(m, n, 11, skip=0.0)
    R = O.restated()
    c = cols.copy(order="F")
    assert R.solve_sweeps_prefix(c, a, d, np.zeros(n + 1), np.zeros(m), step, 1) == 0
    d[step] = 1.0 - 1.0 / R.dot_tree(a[:, step], c[:, step])
    fail, _ = D.solve_sweeps_virtual(cols, a, d, 3, 16, fused=True)
    assert fail == step + 1


@pytest.mark.parametrize("step", [3, 130, 517])
def test_virtual_ranks_breakdown(gpu, step):
    from paper_1502_03543_b200 import dist as D

    m, n = 100, 600
    a, d, cols = _system(m, n, 11, skip=0.0)
    R = O.restated()
    c = cols.copy(order="F")
    assert R.solve_sweeps_prefix(c, a, d, np.zeros(n + 1), np.zeros(m), step, 1) == 0
    d[step] = 1.0 - 1.0 / R.dot_tree(a[:, step], c[:, step])
    ret, _ = _serial(a, d, cols)
    assert ret == step + 1
    fail, _ = D.solve_sweeps_virtual(cols, a, d, 3, 16)
    assert fail == step + 1


@pytest.fixture(scope="module")
def nccl_group(gpu):
    import torch
    import torch.distributed as dist

    if not dist.is_nccl_available():
        pytest.skip("no NCCL")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [0, 3])
def test_solve_lp_group_bitwise(gpu, nccl_group, seed):
    P = gpu
    g = load_golden(f"c1_seed{seed}.npz")
    lp, start = P.gen_random_feasible(50, 200, seed)
    p, st, tr = P.solve_lp(lp, start, group=nccl_group)
    assert st.value == str(g["status"]) and len(tr) == len(g["trace"])
    rows = np.array([[r.gap, r.alpha, r.primal_obj, r.dual_obj, r.r_primal, r.r_dual, r.r_comp,
                      float(r.fallback)] for r in tr])
    assert bits_equal(rows, g["trace"])
    assert bits_equal(p.x, g["x"]) and bits_equal(p.y, g["y"]) and bits_equal(p.s, g["s"])


def test_sharded_solver_c2_first_iterations(gpu, nccl_group):
    """m=500 n=5000 (tile width 16, 40 blocks): side-stream lookahead + NCCL
    broadcasts, two iterations bitwise against the 1-GPU engine."""
    P = gpu
    from paper_1502_03543_b200 import dist as D
    from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver

    lp, start = P.gen_random_feasible(500, 5000, 0)
    outs = []
    for mk in (lambda pr: DeviceSolver(pr), lambda pr: D.ShardedSolver(pr, nccl_group)):
        prob = DeviceProblem.from_lp(lp)
        eng = mk(prob)
        eng.load_iterate(start.x, start.y, start.s)
        sts = [eng.iterate().state for _ in range(2)]
        outs.append(([(s.alpha, s.gap, s.blocking) for s in sts], eng.read_iterate()))
    assert outs[0][0] == outs[1][0]
    for u, v in zip(outs[0][1], outs[1][1]):
        assert bits_equal(u, v)


def test_sharded_solver_peer_exchange(gpu, nccl_group):
    """exchange="peer": [Y | x], workspace and fail word in torch symmetric
    memory (rendezvous over the group), the per-iteration barrier, fused
    panel entry point; two c2 iterations bitwise against the 1-GPU engine."""
    P = gpu
    from paper_1502_03543_b200 import dist as D
    from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver

    lp, start = P.gen_random_feasible(500, 5000, 0)
    outs = []
    for mk in (lambda pr: DeviceSolver(pr),
               lambda pr: D.ShardedSolver(pr, nccl_group, exchange="peer")):
        prob = DeviceProblem.from_lp(lp)
        eng = mk(prob)
        eng.load_iterate(start.x, start.y, start.s)
        sts = [eng.iterate().state for _ in range(2)]
        outs.append(([(s.alpha, s.gap, s.blocking) for s in sts], eng.read_iterate()))
    assert outs[0][0] == outs[1][0]
    for u, v in zip(outs[0][1], outs[1][1]):
        assert bits_equal(u, v)

"""The sharded solve with REAL process separation on one GPU: two processes
(gloo process group, CUDA tensors), each running the CUDA panel / update
blocks of its own shard on cuda:0 and exchanging blocks through
run_collective's broadcasts -- no kernel ever waits on another process, so
sharing one device is safe.  Every rank's solve_lp must equal the 1-GPU
solve bit for bit (trace, iterates), including a trajectory whose cascades
break down and fall back to the direct solve (tests/golden/lp_cases.py), and
the x column rides the x lane on its owner (CudaShard, dist.py)."""

import os
import socket
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _instance(P, case):
    if case[0] == "gen":
        return P.gen_random_feasible(*case[1:])
    sys.path.insert(0, GOLDEN)
    import lp_cases as LC

    A, x, y, s = LC.breakdown_raw(*LC.CASES[case[1]])
    Af = P.DenseMatrix.from_array(np.asfortranarray(A))
    b = np.asarray(P.mat_vec(Af, x))
    c = np.asarray(P.mat_t_vec(Af, y)) + s
    return P.StandardFormLP(Af, b, c), P.InteriorPoint(x, y, s)


def _rows(tr):
    return np.array([[r.gap, r.alpha, r.primal_obj, r.dual_obj, r.r_primal, r.r_dual, r.r_comp,
                      float(r.fallback)] for r in tr])


def _worker(rank, world, port, cases, out_dir):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, REPO)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1502_03543_b200 as P

        for k, (case, max_iter) in enumerate(cases):
            lp, start = _instance(P, case)
            p, st, tr = P.solve_lp(lp, start, P.SolveOptions(max_iter=max_iter),
                                   group=dist.group.WORLD)
            np.savez(os.path.join(out_dir, f"r{rank}_c{k}.npz"), x=p.x, y=p.y, s=p.s,
                     rows=_rows(tr), status=np.array(st.value))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_processes_one_gpu_solve_bitwise(gpu, tmp_path, world):
    import torch.multiprocessing as mp

    P = gpu
    # c: (instance, max_iter); the sharded block is 128 pivots, so n >= 1000
    # gives several blocks per rank; n = 1024 puts x alone in its tile (x lane)
    cases = [(("gen", 300, 1024, 3), 6), (("gen", 200, 1101, 5), 4),
             (("bd", "bd_large"), 14)]
    mp.spawn(_worker, args=(world, _free_port(), cases, str(tmp_path)), nprocs=world,
             join=True)
    for k, (case, max_iter) in enumerate(cases):
        lp, start = _instance(P, case)
        p, st, tr = P.solve_lp(lp, start, P.SolveOptions(max_iter=max_iter))
        want = _rows(tr)
        if case[0] == "bd":
            assert want[:, 7].any()  # the fallback path is exercised
        for r in range(world):
            g = np.load(os.path.join(str(tmp_path), f"r{r}_c{k}.npz"))
            assert str(g["status"]) == st.value, (k, r)
            assert g["rows"].shape == want.shape and np.array_equal(
                g["rows"].view(np.uint64), want.view(np.uint64)), (k, r)
            for name, v in (("x", p.x), ("y", p.y), ("s", p.s)):
                assert np.array_equal(g[name].view(np.uint64), v.view(np.uint64)), (k, r, name)

"""Race stress for the cascade's cross-CTA protocols (release/acquire tile flags,
named barriers, mbarrier rings, the early panel on its own stream, the x lane).

compute-sanitizer is closed on the GPU pool (runs under it left GPUs needing a
reset), so races are hunted the way the pool's policy asks: small cases
repeated many times under perturbed scheduling, every run compared bit for bit
with the CPU oracle.  The perturbation is a competing fp64 workload on a
second stream that occupies a varying number of SMs while the cascade runs,
so panel CTAs, update waves and flag waits interleave differently each time.
"""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

K = O.restated()


def _instance(m, n, seed, breakdown_at=None):
    rng = np.random.default_rng(seed)
    a = np.asfortranarray(rng.uniform(-1, 1, (m, n)))
    cols = np.asfortranarray(rng.uniform(-1, 1, (m, n + 1)) / np.sqrt(m))
    d = np.power(10.0, rng.uniform(-1, 1, n))
    d[rng.random(n) < 0.1] = 1.0
    if breakdown_at is not None:
        c = cols.copy(order="F")
        assert K.solve_sweeps_prefix(c, a, d, np.zeros(n + 1), np.zeros(m), breakdown_at, 1) == 0
        d[breakdown_at] = 1.0 - 1.0 / K.dot_tree(a[:, breakdown_at], c[:, breakdown_at])
    ref = cols.copy(order="F")
    ret = K.solve_sweeps(ref, a, d, np.zeros(n + 1), np.zeros(m), 1)
    return a, cols, d, ref, ret


@pytest.mark.parametrize("m,n,breakdown_at", [
    (50, 300, None), (300, 900, None), (700, 1100, None), (2000, 800, None),
    (300, 1100, 700), (2000, 800, 600),
])
def test_cascade_repeated_under_contention(gpu, m, n, breakdown_at):
    import torch
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200._lib import call, load

    a, cols, d, ref, ret = _instance(m, n, 7 + m, breakdown_at)
    dc0, da, dd = dv.upload(cols), dv.upload(a), dv.upload(d)
    ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8,
                     device=dv.device())
    fail = torch.zeros(1, dtype=torch.int32, device=dv.device())
    noise = torch.cuda.Stream()
    big = torch.rand(2048, 2048, dtype=torch.float64, device=dv.device())
    want = ref.ravel(order="F").view(np.uint64)
    for rep in range(12):
        dc = dc0.clone()
        if rep % 3:
            with torch.cuda.stream(noise):  # competing fp64 work on other SMs
                for _ in range(rep % 3):
                    big = big @ big * 1e-3
        call("pdas_solve_sweeps_ws", dv.ptr(dc), dv.ptr(da), dv.ptr(dd), m, n, dv.ptr(ws),
             rep + 1, dv.ptr(fail), dv.stream())
        torch.cuda.synchronize()
        assert int(fail.item()) == ret, rep
        if ret == 0:
            assert np.array_equal(dv.download(dc).view(np.uint64), want), rep

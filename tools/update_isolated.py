"""The warp-specialized update kernel alone (pdas_cascade_update: one tile per
CTA, 128 pivots) on 148 / 296 / 1480 tiles at m = 2048 and 2000, in cycles per
tile-pivot per wave -- compare with the micro's steady state
(tools/micro/ws2.cu).  profiles/r02_update_isolated.txt.

    python tools/update_isolated.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200._lib import call, load  # noqa: E402
m, n = 2048, 8 * 2000
for m in (2048, 2000):
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    cols = torch.rand(m * (n + 1), dtype=torch.float64, device="cuda", generator=g) * 1e-3
    d = torch.pow(10.0, torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
    ws = torch.zeros(int(load().pdas_cascade_ws_bytes(m, n)), dtype=torch.uint8, device="cuda")
    ws[: n * 8].view(torch.float64)[:] = 1.5  # denominators
    fail = torch.zeros(1, dtype=torch.int32, device="cuda")
    for ntiles in (148, 296, 1480):
        tiles = torch.arange(100, 100 + ntiles, dtype=torch.int64, device="cuda")
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call("pdas_cascade_update", dv.ptr(cols), dv.ptr(A), dv.ptr(d), m, n, 0, 128,
                 dv.ptr(tiles), ntiles, dv.ptr(ws), dv.ptr(fail), torch.cuda.current_stream().cuda_stream)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        waves = (ntiles + 147) // 148
        print(f"m={m} update kernel alone: {ntiles} tiles x 128 pivots: {ms:.3f} ms -> "
              f"{ms * 1e-3 * 1.965e9 / (128 * waves):.0f} cycles per tile-pivot per wave")

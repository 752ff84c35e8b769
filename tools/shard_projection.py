"""Per-rank projection of the column-sharded cascade at G = 1/2/4/8 GPUs from
one GPU (no multi-GPU box in this run).

The sharded schedule (dist.py: block-cyclic pivot blocks of B = 128, chained
or previous-block panels, block broadcasts) is driven over G virtual ranks in lock-step on
the single device, with CUDA events around every panel and update launch of
every rank.  From those device times:

  * work(r)   = sum of rank r's panel + update kernel times (what rank r's GPU
                would be busy with);
  * chain     = sum over blocks of the panel times (panel b+1 can only start
                once block b is final and broadcast: the serial spine), plus,
                for the chained schedule (default), one update CTA-duration per
                block (the panel waits for its own tiles' update);
  * exchange  = blocks x (an NVLink broadcast of the block's B*m*8 bytes at
                --nvlink-gbs plus --bcast-us of NCCL latency).

projected time per cascade ~ max(max_r work(r), chain + exchange).  Printed
with the inputs, so DESIGN.md §6 can quote it; it is a model, not a
measurement.

    python tools/shard_projection.py [--m 2000 --n 20000] [--gpus 1,2,4,8]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_03543_b200 import _device as dv  # noqa: E402
from paper_1502_03543_b200 import dist as D  # noqa: E402
from paper_1502_03543_b200._lib import load  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2000)
ap.add_argument("--n", type=int, default=20000)
ap.add_argument("--gpus", default="1,2,4,8")
ap.add_argument("--nvlink-gbs", type=float, default=600.0,
                help="effective per-broadcast NVLink bandwidth (GB/s)")
ap.add_argument("--bcast-us", type=float, default=25.0, help="NCCL latency per broadcast")
ap.add_argument("--previous-block", action="store_true",
                help="the r01 schedule (panels apply the previous block) instead of the chained one")
args = ap.parse_args()
m, n = args.m, args.n


class TimedShard(D.CudaShard):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.ev = []  # (kind, block, start event, end event)

    def _timed(self, kind, b, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        self.ev.append((kind, b, e0, e1))

    def panel(self, q0, p0, p1, tag=0):
        self._timed("panel", p0 // self.plan.B,
                    lambda: super(TimedShard, self).panel(q0, p0, p1, tag=tag))

    def update(self, p0, p1, i0, tag=0):
        self._timed("update", p0 // self.plan.B,
                    lambda: super(TimedShard, self).update(p0, p1, i0, tag=tag))


g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.rand(m * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
cols0 = torch.rand(m * (n + 1), dtype=torch.float64, device="cuda", generator=g) * 1e-3
d = torch.pow(10.0, torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1)
wsb = int(load().pdas_cascade_ws_bytes(m, n))
print(f"m={m} n={n}: sharded cascade (B={D.cascade_block_pivots()}, tile "
      f"{D.cascade_tile_width(m)}, {'previous-block' if args.previous_block else 'chained'} "
      f"panels), lock-step virtual ranks on one B200; model inputs "
      f"nvlink {args.nvlink_gbs:.0f} GB/s, {args.bcast_us:.0f} us/broadcast")
print("   G   work/rank max ms   work/rank min ms   panel chain ms   exchange ms   "
      "projected ms   vs G=1")
base = None
for G in [int(x) for x in args.gpus.split(",")]:
    plans = [D.make_plan(m, n, G, r) for r in range(G)]
    bufs = [(cols0.clone(), torch.zeros(wsb, dtype=torch.uint8, device="cuda"),
             torch.zeros(1, dtype=torch.int32, device="cuda")) for _ in range(G)]
    bes = [TimedShard(plans[r], bufs[r][0], A, d, bufs[r][1], bufs[r][2], streams=False)
           for r in range(G)]
    for be in bes:
        be.chained = not args.previous_block
    for rep in range(2):  # warm-up + measured
        for be, (c, _, f) in zip(bes, bufs):
            c.copy_(cols0)
            f.zero_()
            be.ev.clear()
        D.run_lockstep(plans, bes)
        torch.cuda.synchronize()
    work = [sum(e0.elapsed_time(e1) for _, _, e0, e1 in be.ev) for be in bes]
    chain = sum(e0.elapsed_time(e1) for be in bes for kind, _, e0, e1 in be.ev
                if kind == "panel")
    nb = plans[0].nb
    if not args.previous_block:
        # chained: each panel also waits for its rank's update of the block's own
        # tiles -- one CTA-duration of an update, ~ the shortest update launch
        one_wave = min(e0.elapsed_time(e1) for be in bes for kind, _, e0, e1 in be.ev
                       if kind == "update")
        chain += (nb - 1) * one_wave
    blk_bytes = plans[0].B * m * 8
    exch = 0.0 if G == 1 else nb * (blk_bytes / (args.nvlink_gbs * 1e9) * 1e3 +
                                    2 * args.bcast_us * 1e-3)
    proj = max(max(work), chain + exch)
    base = base or proj
    print(f"{G:4d} {max(work):18.1f} {min(work):18.1f} {chain:16.1f} {exch:13.1f} "
          f"{proj:14.1f} {base / proj:7.2f}x")
    del bufs, bes
    torch.cuda.empty_cache()

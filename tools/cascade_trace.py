"""Per-phase cycle breakdown of the update kernel (block 20, CTA 0, warps 0
and last) from the clock64 trace (PDAS_CASCADE_MODE=3)."""
import ctypes
import os
import subprocess
import sys

os.environ["PDAS_CASCADE_MODE"] = "3"
sys.argv = [sys.argv[0], "--reps", "1"]
here = os.path.dirname(os.path.abspath(__file__))
exec(open(os.path.join(here, "cascade_time.py")).read())
from paper_1502_03543_b200._lib import load  # noqa: E402

buf = (ctypes.c_longlong * 192)()
load().pdas_debug_cascade_trace(buf, 192)
names = ["wait_full", "partials", "B1+producer", "reduce+B2", "axpy"]
for slot in range(2):
    tot = [0] * 5
    for j in range(16):
        t = [buf[(slot * 16 + j) * 6 + k] for k in range(6)]
        d = [t[k + 1] - t[k] for k in range(5)]
        tot = [a + b for a, b in zip(tot, d)]
    print(f"warp slot {slot}: avg cycles per pivot: " +
          ", ".join(f"{n}={v / 16:.0f}" for n, v in zip(names, tot)) + f", total={sum(tot) / 16:.0f}")

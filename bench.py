"""Benchmark: PDAS iterations/s at m=2000, n=20000 (BASELINE.json configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one full PDAS iteration (solver.py:222-278) of the seeded LP
gen_random_feasible(2000, 20000, 0): scaling, A x, x0 = L0^-T L0^-1 A x, the
Egidi-Maponi cascade over [Y | x] (20000 rank-one steps), A^T dy, residuals,
ratio test, x/y/s update, gap and objectives.  Every step restarts from the
generator's start point so all K steps do identical work.  The one-time
prepare (gram, Cholesky, Y) is timed and reported separately.

Prints ONE JSON line (rank 0).  See DESIGN.md §5 for every field.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

M, N, SEED = 2000, 20000, 0
METRIC = "PDAS iterations/s (m=2000, n=20000)"
# identical in both arms (driver: same_config); what runs where goes in the
# top-level "parallelism" / "cascade" keys
CONFIG = {"workload": f"c3 dense LP m={M} n={N} seed={SEED} (BASELINE configs[2]), each step = "
                      "PDAS iteration 1 from the generator's start", "m": M, "n": N,
          "l2": "no flush: inputs larger than L2 ([Y|x] 320 MB + A 320 MB + Y 320 MB)"}
UNIT = "iterations/s"


def algorithmic(m, n):
    """Per cascade: element-steps E, streaming bytes (16 B per element-step +
    pivot/A columns) and fp64 operations (4 per element-step)."""
    E = m * n * (n + 1) // 2
    return E, 16 * E + 16 * m * n, 4 * E


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """One `nvidia-smi --query-gpu ... -lms 200` process for the whole timed
    region (B200_PROFILING.md clocks line); parsed afterwards."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.path = os.path.join(REPO, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.fh.close()
            for line in open(self.path):
                parts = [x.strip() for x in line.strip().split(",")]
                if len(parts) >= 8:
                    self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU legs
def cascade_traffic(n, block=256):
    """DRAM bytes (read + write) of one c3 cascade, from the committed ncu
    launch list of `tools/cascade_time.py` (profiles/r02_launches_cascade.json:
    per-kernel sums of dram__bytes_read.sum + dram__bytes_write.sum).  One
    panel launch per pivot block: the first block has `block` pivots, the
    others 2 * block (cascade.cu run_cascade_impl)."""
    try:
        d = json.load(open(os.path.join(REPO, "profiles", "r02_launches_cascade.json")))
    except Exception:
        return None
    casc = {k: v for k, v in d.items() if "k_casc" in k}
    panels = sum(v["launches"] for k, v in casc.items() if "panel" in k)
    if not panels:
        return None
    blocks = 1 + max(0, (n - block + 2 * block - 1) // (2 * block))
    ncasc = panels / blocks
    return sum(v["dram_bytes"] for v in casc.values()) / ncasc


def cpu_cascade_sample(a, y, x0col, d, steps, threads):
    """Time the reference's compiled core (oracle/_ref, else the restated
    oracle) on cascade steps [0, steps) of the c3 workload; returns
    (seconds, element-steps, kind)."""
    from oracle import oracle as O

    k = O.reference()
    kind = "reference" if k is not None else "port"
    k = k or O.restated()
    m, n = a.shape
    cols = np.empty((m, n + 1), order="F")
    cols[:, :n] = y
    cols[:, n] = x0col
    dd = np.where(np.arange(n) < steps, d, 1.0)
    t0 = time.perf_counter()
    k.solve_sweeps(cols, a, dd, np.zeros(n + 1), np.zeros(m), threads)
    dt = time.perf_counter() - t0
    es = sum(m * (n + 1 - l) for l in range(steps))
    return dt, es, kind


def cpu_rate(dt, es, m, n):
    """iterations/s extrapolated from a cascade sample (the cascade is >99 %
    of an iteration)."""
    E, _, _ = algorithmic(m, n)
    return 1.0 / (dt / es * E)


def host_inputs():
    """c3 instance + d of iteration 1 on the host, without any GPU code:
    numpy RNG (the generator's draw order) and LAPACK for Y / x0 (untimed
    setup of the CPU sample; only the sample's timing is reported)."""
    rng = np.random.default_rng(SEED)
    a = np.asfortranarray(rng.uniform(-1.0, 1.0, size=(M, N)))
    x = rng.uniform(0.5, 2.0, size=N)
    s = rng.uniform(0.5, 2.0, size=N)
    g = a @ a.T
    y = np.asfortranarray(np.linalg.solve(g, a))
    x0col = np.linalg.solve(g, a @ x)
    return a, y, x0col, x / s


def run_reference(args):
    """--impl reference: the reference's own compiled CPU core on this host,
    all host threads.  Each of the W + K steps is a bounded sample (cascade
    steps 0..S-1 of iteration 1, the >99 % part of an iteration); after them
    ONE full 20000-step cascade of iteration 1 is timed as well.  `value` is
    the full cascade's rate (measured, not extrapolated; the rest of a
    reference iteration is ~0.05 s); `ms_per_step` is what each
    sample step really took, so steps x ms_per_step is the timed work."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    a, y, x0col, d = host_inputs()
    steps = args.ref_sample_steps
    rates, times = [], []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        dt, es, kind = cpu_cascade_sample(a, y, x0col, d, steps, threads)
        if i >= args.warmup:
            rates.append(cpu_rate(dt, es, M, N))
            times.append(dt)
    sample_rate = float(np.median(rates))
    full_s = None
    if not args.ref_no_full:
        full_s, _, kind = cpu_cascade_sample(a, y, x0col, d, N, threads)
    value = 1.0 / full_s if full_s else sample_rate
    sample = (f"each step: cascade steps 0..{steps - 1} of PDAS iteration 1 at m={M}, n={N} "
              f"(d = x0/s0); value: one full {N}-step cascade of that iteration, timed "
              f"({full_s:.1f} s)" if full_s else "value extrapolated by element-steps")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.median(times)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(CONFIG), "parallelism": f"CPU, {threads} threads (OpenMP)",
        "step": f"bounded sample: cascade steps 0..{steps - 1} (not a whole iteration)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample, "full_cascade_s": full_s,
                         "sample_extrapolated_value": sample_rate,
                         "sample_seconds": float(np.median(times))},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PDAS_BENCH_BACKEND=gloo runs the N > 1 code path with several ranks on one
    # GPU (a functional check of the sharded bench; timings are meaningless)
    backend = os.environ.get("PDAS_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_1502_03543_b200 as P
    from paper_1502_03543_b200 import _device as dv
    from paper_1502_03543_b200._lib import call, load as load_lib
    from paper_1502_03543_b200.engine import DeviceProblem, DeviceSolver

    shard = world > 1 and args.mode == "shard"
    # instance (identical bits to the reference generator) + one-time prepare
    lp, start = P.gen_random_feasible(M, N, SEED)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = DeviceProblem.from_lp(lp)
    L0 = prob.validate()
    if shard:
        from paper_1502_03543_b200.dist import ShardedSolver

        eng = ShardedSolver(prob, dist.group.WORLD, 0.9, L0=L0, exchange=args.exchange)
    else:
        eng = DeviceSolver(prob, "woodbury", 0.9, L0=L0)
    torch.cuda.synchronize()
    prepare_s = time.perf_counter() - t0

    x0 = dv.upload(start.x)
    y0 = dv.upload(start.y)
    s0 = dv.upload(start.s)

    def reset():
        eng.x.copy_(x0)
        eng.y.copy_(y0)
        eng.s.copy_(s0)

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        reset()
        eng.iterate()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = eng.launches
    if not shard:
        eng.time_cascade = True  # events around the cascade inside each timed step
        eng.cascade_events.clear()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            reset()
            res = eng.iterate()
        ev1.record(stream)
        torch.cuda.synchronize()
    casc_in_step = [a.elapsed_time(b) for a, b in getattr(eng, "cascade_events", [])]
    if not shard:
        eng.time_cascade = False
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = (eng.launches - launches0) // max(args.steps, 1)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    # shard: one LP over all ranks; replicas: iterations/s summed over ranks
    jobs = 1 if shard else world
    value = jobs * 1e3 / ms_per_step

    # ---- the dominant kernels' time: the cascade (x0 lane + panels + updates,
    # pdas_solve_sweeps_ws_x0) timed with CUDA events on the solver's stream
    # INSIDE the timed steps above
    m, n = M, N
    if casc_in_step:
        casc_s = float(np.median(casc_in_step)) / 1e3
        casc_src = (f"median over the {len(casc_in_step)} timed steps: events around "
                    "pdas_solve_sweeps_ws_x0 inside DeviceSolver.iterate")
    else:  # sharded: the per-rank cascade is not one launch sequence
        casc_s = ms_per_step / 1e3
        casc_src = "sharded run: whole step"
    d_it1 = eng.d.clone()  # d of iteration 1 (x0/s0), for the CPU sample
    xcol0 = eng.rhs.clone()  # x0 = L0^-T L0^-1 (A x0)
    from paper_1502_03543_b200.engine import d_solve_many

    d_solve_many(eng.basis.L0, m, xcol0, 1)
    E, Bytes, Flops = algorithmic(m, n)
    # fp64 (separate mul/add) peak of this GPU, measured now
    sink = dv.empty(1)
    ops = __import__("ctypes").c_int64()
    call("pdas_probe_fp64", dv.ptr(sink), 20000, __import__("ctypes").addressof(ops),
         stream.cuda_stream)
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    call("pdas_probe_fp64", dv.ptr(sink), 20000, __import__("ctypes").addressof(ops),
         stream.cuda_stream)
    p1.record(stream)
    torch.cuda.synchronize()
    fp64_peak = ops.value / (p0.elapsed_time(p1) / 1e3) / 1e12
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved_tf = Flops / casc_s / 1e12
    roofline = {
        "bound": "fp64", "achieved": achieved_tf, "peak": fp64_peak, "unit": "TFLOP/s",
        "frac": achieved_tf / fp64_peak, "traffic": cascade_traffic(N),
        "traffic_unit": "bytes per cascade (DRAM read+write of all k_casc_* launches, ncu)",
        "traffic_source": "STATIC: read from the committed ncu launch list "
                          "profiles/r02_launches_cascade.json (not measured in this run)",
        "kernel": "cascade (k_casc_panel + k_casc_update), one 20000-step solve",
        "peak_source": "measured now: pdas_probe_fp64 (separate DMUL+DADD, no FMA)",
        "hbm_equivalent": {
            "achieved": Bytes / casc_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": Bytes / casc_s / 1e9 / hbm_peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
            "note": "algorithmic bytes of the one-pass streaming cascade (16 B per "
                    "element-step + pivot/A columns); frac > 1 = the register-tiled "
                    "schedule moves less than the streaming minimum"},
        "cascade_ms": casc_s * 1e3,
        "cascade_ms_source": casc_src,
    }

    # ---- e2e through the public API: host iterate in, host iterate out
    hx = torch.from_numpy(start.x.copy()).pin_memory()
    hy = torch.from_numpy(start.y.copy()).pin_memory()
    hs = torch.from_numpy(start.s.copy()).pin_memory()
    ox, oy, os_ = (torch.empty_like(t).pin_memory() for t in (hx, hy, hs))
    e2e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.load_iterate(hx, hy, hs)
        eng.iterate()
        ox.copy_(eng.x, non_blocking=True)
        oy.copy_(eng.y, non_blocking=True)
        os_.copy_(eng.s, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    h2d = 8 * (2 * N + M)
    d2h = 8 * (2 * N + M) + 104

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(CONFIG),
        "parallelism": (f"column-sharded cascade over {world} GPUs (dist.py, "
                        f"{args.exchange} block exchange)" if shard
                        else f"replicas x{world}" if world > 1 else "1 GPU"),
        "cascade_block_pivots": (int(load_lib().pdas_cascade_block_pivots()) if shard
                                 else f"{int(load_lib().pdas_cascade_solve_block())} then "
                                      f"{2 * int(load_lib().pdas_cascade_solve_block())}"),
        "e2e": {"value": jobs / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "roofline": roofline,
        "prepare_s": prepare_s,
        "alpha_it1": res.state.alpha,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        # cpu_baseline: bounded sample of the same workload on this host
        a = lp.A.as_2d()
        yb = dv.download(eng.basis.Y).reshape((M, N), order="F")
        threads = os.cpu_count() or 1
        dt, es, kind = cpu_cascade_sample(a, yb, dv.download(xcol0), dv.download(d_it1),
                                          args.cpu_sample_steps, threads)
        line["cpu_baseline"] = {
            "value": cpu_rate(dt, es, M, N), "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"cascade steps 0..{args.cpu_sample_steps - 1} of iteration 1 "
                      f"({dt:.1f} s), extrapolated by element-steps to the full cascade"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-steps", type=int, default=1500)
    ap.add_argument("--ref-sample-steps", type=int, default=1000)
    ap.add_argument("--ref-no-full", action="store_true",
                    help="reference arm: skip the one full-cascade timing")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="shard", choices=["shard", "replicas"],
                    help="N>1: one LP column-sharded over the GPUs, or N independent LPs")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="shard mode: NCCL broadcast per pivot block, or the panel's fused "
                         "NVLink peer stores")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

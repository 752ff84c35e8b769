"""Verification and benchmark harnesses on the GPU, plus an instance cache.

Mirrors the reference's `adascale check` / `adascale bench` (cli.py:144-217,
random_system :165-180) on this package's device path -- SURVEY.md §8(f)
rows 3 and 4.  The rest of the reference CLI (solve / gen front end, JSON
files, exit-code plumbing of `solve`) is out of scope.

    python -m paper_1502_03543_b200 check [--seeds 1..20] [--m M --n N]
                                          [--z-tol 1e-9] [--equiv-tol 1e-8]
    python -m paper_1502_03543_b200 bench --grid 50x200,500x5000 [--max-iter 20]

`check` exits 5 when a threshold is exceeded (cli.py:26-37, EXIT_CHECK_FAILED),
2 on bad arguments.  The Woodbury-vs-direct gap it reports is bit-identical
to the reference's (both solves are); the Z-residual comes from cuBLAS
products instead of the reference's numpy BLAS, so it agrees to rounding.
"""

from __future__ import annotations

import hashlib
import math
import os
import time
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import GenerationError, NotPositiveDefinite
from .linalg import DenseMatrix, cholesky_factor, gram
from .model import InteriorPoint, StandardFormLP, gen_random_feasible
from .normal import prepare_woodbury, solve_direct, solve_woodbury
from .solver import SolveOptions, solve_lp, z_inverse_check

EXIT_OK, EXIT_USAGE, EXIT_CHECK_FAILED = 0, 2, 5


def parse_seed_range(text: str) -> List[int]:
    """cli.py:82-95: "N" or "A..B" (inclusive)."""
    if ".." in text:
        lo_text, hi_text = text.split("..", 1)
        try:
            lo, hi = int(lo_text), int(hi_text)
        except ValueError:
            raise ValueError(f"seed range '{text}' is not of the form A..B") from None
        if hi < lo:
            raise ValueError(f"seed range '{text}' is empty")
        return list(range(lo, hi + 1))
    try:
        return [int(text)]
    except ValueError:
        raise ValueError(f"seeds must be an integer or A..B range, got '{text}'") from None


def random_system(rng, m: int, n: int) -> Tuple[DenseMatrix, np.ndarray, np.ndarray]:
    """cli.py:165-180: full-rank A ~ U[-1,1] (redrawn until chol(gram(A))
    passes, on the GPU), d = 10^U[-3,3], rhs ~ U[-1,1] -- the reference's
    draw order, so the same seed gives the same system."""
    a = None
    for _ in range(100):
        cand = DenseMatrix.from_array(rng.uniform(-1.0, 1.0, size=(m, n)))
        try:
            cholesky_factor(gram(cand))
        except NotPositiveDefinite:
            continue
        a = cand
        break
    if a is None:
        raise GenerationError("no full-rank draw in 100 attempts")
    d = np.power(10.0, rng.uniform(-3.0, 3.0, size=n))
    rhs = rng.uniform(-1.0, 1.0, size=m)
    return a, d, rhs


def check_system(seed: int, m: Optional[int] = None, n: Optional[int] = None):
    """One seed of run_check (cli.py:188-209): (m, n, z_residual, gap, w_direct,
    w_woodbury)."""
    rng = np.random.default_rng(seed)
    m = m if m is not None else int(rng.integers(1, 6))
    n = n if n is not None else int(rng.integers(m + 1, 9))
    if not 1 <= m <= n:
        raise ValueError(f"check needs 1 <= m <= n, got m={m}, n={n}")
    if m == 1 and n == 1:  # the hand-verified self-check system
        a = DenseMatrix.from_rows([[2.0]])
        d = np.array([3.0])
        rhs = np.array([6.0])
    else:
        a, d, rhs = random_system(rng, m, n)
    z_res = z_inverse_check(a, d)
    w_direct = solve_direct(a, d, rhs)
    w_wood = solve_woodbury(prepare_woodbury(a), a, d, rhs)
    gap = float(np.max(np.abs(w_wood - w_direct))) / (1.0 + float(np.max(np.abs(w_direct))))
    return m, n, z_res, gap, w_direct, w_wood


def run_check(seeds: Sequence[int], m: Optional[int] = None, n: Optional[int] = None,
              z_tol: float = 1e-9, equiv_tol: float = 1e-8, out=print) -> int:
    """cli.py:183-217 on the GPU: max Z-residual and max backend gap over the
    seeds; exit 5 if either threshold is exceeded."""
    if z_tol <= 0 or equiv_tol <= 0:
        raise ValueError("check tolerances must be positive")
    max_z = max_gap = 0.0
    offending = []
    for seed in seeds:
        _, _, z_res, gap, _, _ = check_system(seed, m, n)
        max_z = max(max_z, z_res)
        max_gap = max(max_gap, gap)
        if z_res > z_tol or gap > equiv_tol:
            offending.append(seed)
    out(f"max Z-residual {max_z!r}, max backend gap {max_gap!r}")
    if offending:
        out(f"thresholds exceeded for seeds: {','.join(str(s) for s in offending)}")
        return EXIT_CHECK_FAILED
    return EXIT_OK


def parse_grid(text: str) -> List[Tuple[int, int]]:
    out = []
    for item in text.split(","):
        try:
            m, n = item.lower().split("x")
            out.append((int(m), int(n)))
        except ValueError:
            raise ValueError(f"grid entry '{item}' is not of the form MxN") from None
    return out


def run_bench(grid: Sequence[Tuple[int, int]], seed: int = 0, max_iter: int = 20,
              workers: Sequence[int] = (1,), out=print) -> List[str]:
    """cli.py:144-162: CSV m,n,backend,workers,iterations,ms_per_iter of
    solve_lp over a grid (GPU; `workers` is accepted for the same columns)."""
    from .errors import AdascaleError

    rows = ["m,n,backend,workers,iterations,ms_per_iter"]
    out(rows[0])
    for m, n in grid:
        lp, start = gen_random_feasible(m, n, seed)
        for backend in ("direct", "woodbury"):
            for w in workers:
                opts = SolveOptions(backend=backend, workers=w, max_iter=max_iter)
                try:
                    t0 = time.perf_counter()
                    _, _, trace = solve_lp(lp, start, opts)
                    elapsed = (time.perf_counter() - t0) * 1e3
                    iters = len(trace)
                    per = elapsed / iters if iters else math.nan
                except AdascaleError:
                    iters, per = 0, math.nan
                rows.append(f"{m},{n},{backend},{w},{iters},{per:.3f}")
                out(rows[-1])
    return rows


# ------------------------------------------------------------------ instance cache
def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def cached_instance(m: int, n: int, seed: int,
                    cache_dir: Optional[str] = None) -> Tuple[StandardFormLP, InteriorPoint]:
    """gen_random_feasible(m, n, seed) through an on-disk .npz cache (c3's A is
    320 MB and c4's 800 MB; the draw + rank check + A x / A^T y are paid once).
    The file stores A column-major plus b, c, x, y, s and a sha256 of A; a
    stale or corrupt file is regenerated.  cache_dir defaults to
    $PDAS_INSTANCE_CACHE or ~/.cache/pdas_b200."""
    cache_dir = cache_dir or os.environ.get("PDAS_INSTANCE_CACHE") or os.path.join(
        os.path.expanduser("~"), ".cache", "pdas_b200")
    path = os.path.join(cache_dir, f"lp_m{m}_n{n}_s{seed}.npz")
    if os.path.exists(path):
        try:
            z = np.load(path, allow_pickle=False)
            a = np.asarray(z["A"])
            if a.shape == (m * n,) and str(z["A_sha"]) == _sha(a):
                lp = StandardFormLP(DenseMatrix(m, n, a), z["b"], z["c"])
                return lp, InteriorPoint(z["x"], z["y"], z["s"])
        except Exception:
            pass
    lp, start = gen_random_feasible(m, n, seed)
    os.makedirs(cache_dir, exist_ok=True)
    tmp = path + f".tmp{os.getpid()}.npz"
    np.savez(tmp, A=lp.A.data, A_sha=np.array(_sha(lp.A.data)), b=lp.b, c=lp.c, x=start.x,
             y=start.y, s=start.s)
    os.replace(tmp, path)
    return lp, start

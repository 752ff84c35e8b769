"""Deterministic column partitioning of the sweep.

Mirrors adascale/parallel.py.  In the reference, `workers` CPU threads split
the live columns of each step into contiguous ranges (column_partition,
:59-78) and run the two sweep phases with a join barrier (:94-166); results
are bitwise identical for every worker count.  On B200 the same independence
is exploited by CTAs (register tiles of columns, cascade.cu) and by GPUs
(column-cyclic shards, dist.py), so `workers` no longer selects an engine: it
is validated and recorded, and every path below runs the CUDA cascade.
The partition helpers are kept verbatim in meaning -- dist.py reuses the
same plan vocabulary for its shard map.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Dict, Optional, Tuple

import numpy as np

from .errors import DimensionMismatch
from .linalg import DenseMatrix, as_vector
from .normal import AugWorkspace, WoodburyBasis, rank_one_step, solve_woodbury


def resolve_workers(workers: int) -> int:
    """0 means all cores (parallel.py:27-33)."""
    if workers < 0:
        raise ValueError(f"workers must be >= 0, got {workers}")
    if workers == 0:
        return os.cpu_count() or 1
    return workers


@dataclass(frozen=True)
class SweepPlan:
    """Static column assignment for one step; depends only on (n, workers, l)."""

    assignments: Dict[int, Tuple[int, int]]
    workers: int
    phase_barriers: int = 2

    def phase1_range(self, worker: int) -> Tuple[int, int]:
        return self.assignments[worker]

    def phase2_range(self, worker: int, l: int) -> Tuple[int, int]:
        """Phase-1 range with the frozen pivot column clipped out."""
        k0, k1 = self.assignments[worker]
        return max(k0, l), k1

    def active_columns(self) -> set:
        cover = set()
        for k0, k1 in self.assignments.values():
            cover.update(range(k0, k1))
        return cover


def column_partition(ncols: int, workers: int, l: int) -> SweepPlan:
    """Live columns l-1 .. ncols (incl. the solution column) of step l in
    ceil(active/workers)-sized contiguous ranges (parallel.py:59-78)."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if not 1 <= l <= ncols:
        raise DimensionMismatch(f"step index {l} outside 1..{ncols}")
    lo, hi = l - 1, ncols + 1
    chunk = -(-(hi - lo) // workers)
    assignments = {}
    for w in range(workers):
        k0 = min(lo + w * chunk, hi)
        assignments[w] = (k0, min(k0 + chunk, hi))
    return SweepPlan(assignments, workers)


@dataclass(frozen=True)
class ParamContext:
    """Per-sweep parameters (parallel.py:81-91)."""

    m: int
    n: int
    l: int
    d_l: float
    cols: np.ndarray
    inner: np.ndarray
    v_scratch: np.ndarray


def parallel_sweep(ws: AugWorkspace, a: DenseMatrix, d, l: int, workers: int,
                   pool=None) -> AugWorkspace:
    """Rank-one step l, bitwise identical to `rank_one_step` for any `workers`
    (parallel.py:94-139); the column split happens inside the CUDA kernels."""
    resolve_workers(workers)
    d = as_vector(d, "d")
    return rank_one_step(ws, a, d, l)


def solve_woodbury_parallel(basis: WoodburyBasis, a: DenseMatrix, d, b, workers: int,
                            pool: Optional[object] = None) -> np.ndarray:
    """Full cascade solve; bitwise identical to `solve_woodbury` (parallel.py:169-209)."""
    d = as_vector(d, "d")
    b = as_vector(b, "b")
    if basis.m != a.rows or basis.n != a.cols:
        raise DimensionMismatch("basis does not match the matrix")
    if d.size != a.cols or b.size != a.rows:
        raise DimensionMismatch("scaling or rhs length does not match the matrix")
    if d.size and float(np.min(d)) <= 0.0:
        raise ValueError("solve requires strictly positive scaling entries")
    resolve_workers(workers)
    return solve_woodbury(basis, a, d, b)

"""Seeded LPs that drive solve_lp into the reference's rare exits (numpy only,
so the golden generator and the GPU tests build bit-identical instances).

breakdown_lp(m, n, l, seed, dl, dscale)
    Row 0 of A is e_l (A[0, l] = 1, zero elsewhere), so column l's leverage
    a_l^T M^{-1} a_l is exactly 1 and the cascade's step l sees
    denom = 1 + (d_l - 1) * 1 = d_l (breakdown is d_l -> 0 with
    a_l^T M^{-1} a_l -> 1).  The start has d = x/s ~ dscale everywhere and
    d_l = dl:
      * dl = 1e-13, dscale = 1e-12: |denom| <= 1e-12 (1 + |inner|) -> the
        cascade returns l+1 -> SingularUpdate -> solve_direct (solver.py:161-165),
        whose Cholesky passes (its eps is relative to max diag(A D A^T) ~ 1e-11)
        -> a trajectory with fallback=True rows;
      * dl = 1e-14, dscale = 1e-3: the fallback's Cholesky fails too
        (diag 1e-14 < 1e-12 * max diag) -> NUMERICAL_BREAKDOWN (solver.py:226-228).
    b = A x and c = A^T y + s make the start exactly feasible (model.py:122-131).
"""

import numpy as np


def breakdown_raw(m, n, l, seed, dl, dscale):
    """(A (m x n, C order), x, y, s) before b and c are formed."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, (m, n))
    A[0, :] = 0.0
    A[0, l] = 1.0
    x = rng.uniform(0.5, 2.0, n) * np.sqrt(dscale)
    s = rng.uniform(0.5, 2.0, n) / np.sqrt(dscale)
    x[l] = np.sqrt(dl)
    s[l] = 1.0 / np.sqrt(dl)
    y = rng.uniform(-1.0, 1.0, m)
    return A, x, y, s


# (tag, m, n, l, seed, dl, dscale): bd_* fall back and converge, nb_* break down
CASES = {
    "bd_small": (20, 60, 7, 0, 1e-13, 1e-12),
    "bd_large": (300, 3000, 700, 1, 1e-13, 1e-12),
    "nb_small": (20, 60, 7, 0, 1e-14, 1e-3),
}

"""The drop-in boundary, exercised from the reference's side.

The UNMODIFIED reference Python package (staged by oracle/build_ref.sh into
the git-ignored oracle/_ref/pkg/adascale, next to its compiled core) is
imported with its kernel core swapped for this repo's B200 table exactly as
INTEGRATION.md §2 tells a maintainer to do it: the module object
`adascale._core.kernels` (_core.py:10-16) and the names the callers bound at
import time (linalg.py:14, normal.py:24, parallel.py:21).  The reference's own
gen_random_feasible and solve_lp then run with every kernel call (tree dots,
mat_vec, gram, Cholesky, solves, the cascade) on the GPU, and must land on the
reference's golden bits (c1 seed 0: 25 iterations, OPTIMAL)."""

import importlib
import os
import sys

import numpy as np
import pytest

from conftest import REPO, bits_equal, load_golden, sha

pytestmark = pytest.mark.gpu

STAGED = os.path.join(REPO, "oracle", "_ref", "pkg")


@pytest.fixture(scope="module")
def ref_on_b200(gpu):
    if not os.path.isfile(os.path.join(STAGED, "adascale", "solver.py")):
        pytest.fail("oracle/_ref/pkg not staged: run `make -C oracle` (oracle/build_ref.sh)")
    saved = {k: v for k, v in sys.modules.items() if k == "adascale" or k.startswith("adascale.")}
    for k in saved:
        del sys.modules[k]
    old_env = os.environ.get("ADASCALE_PURE_PYTHON")
    os.environ["ADASCALE_PURE_PYTHON"] = "1"  # import without the CPU core ...
    sys.path.insert(0, STAGED)
    try:
        ad = importlib.import_module("adascale")
        from paper_1502_03543_b200._core import kernels as b200

        # ... then bind the B200 table where the reference looks it up
        for name in ("_core", "linalg", "normal", "parallel"):
            setattr(sys.modules[f"adascale.{name}"], "kernels", b200)
        assert ad.active_core() == "compiled"  # the table reports COMPILED = True
        yield ad
    finally:
        sys.path.remove(STAGED)
        for k in [k for k in sys.modules if k == "adascale" or k.startswith("adascale.")]:
            del sys.modules[k]
        sys.modules.update(saved)
        if old_env is None:
            os.environ.pop("ADASCALE_PURE_PYTHON", None)
        else:
            os.environ["ADASCALE_PURE_PYTHON"] = old_env


def test_reference_solve_lp_over_b200_kernels(ref_on_b200):
    ad = ref_on_b200
    assert ad.linalg.kernels.__class__.__name__ == "_CudaKernels"
    g = load_golden("c1_seed0.npz")
    lp, start = ad.gen_random_feasible(50, 200, 0)
    assert sha(lp.A.data) == str(g["A_sha"])
    assert bits_equal(lp.b, g["b"]) and bits_equal(lp.c, g["c"])
    p, st, tr = ad.solve_lp(lp, start)
    assert st.value == str(g["status"]) == "optimal" and len(tr) == len(g["trace"]) == 25
    rows = np.array([[r.gap, r.alpha, r.primal_obj, r.dual_obj, r.r_primal, r.r_dual, r.r_comp,
                      float(r.fallback)] for r in tr])
    assert bits_equal(rows, g["trace"])
    assert bits_equal(p.x, g["x"]) and bits_equal(p.y, g["y"]) and bits_equal(p.s, g["s"])


def test_reference_layers_over_b200_kernels(ref_on_b200):
    """The reference's L2/L3 wrappers (linalg, normal) on the B200 table:
    prepare_woodbury, init_workspace + rank_one_step chain vs the golden basis."""
    ad = ref_on_b200
    g = load_golden("c1_seed0.npz")
    lp, _ = ad.gen_random_feasible(50, 200, 0)
    basis = ad.prepare_woodbury(lp.A)
    assert bits_equal(basis.L0.as_2d(), g["L0"]) and bits_equal(basis.Y.as_2d(), g["Y"])
    ws = ad.init_workspace(basis, g["it1_rhs"])
    assert bits_equal(ws.cols[:, -1], g["it1_x0col"])
    dy = ad.solve_woodbury(basis, lp.A, g["it1_d"], g["it1_rhs"])
    assert bits_equal(dy, g["it1_dy"])

"""Host-side logic that needs no GPU: option validation, containers, the
error taxonomy, partition semantics, JSON I/O, and the loud failure when no
CUDA device exists (no CPU fallback)."""

import numpy as np
import pytest

import paper_1502_03543_b200 as P
from paper_1502_03543_b200 import _lib


def test_public_surface_mirrors_reference():
    # adascale/__init__.py:66-114
    expected = {
        "AdascaleError", "AugWorkspace", "DenseMatrix", "DimensionMismatch", "Directions",
        "GenerationError", "InteriorPoint", "LowerTriangular", "NonFiniteEntry", "NotFeasible",
        "NotInterior", "NotPositiveDefinite", "RankDeficient", "SchemaError", "SingularUpdate",
        "SolveOptions", "StandardFormLP", "Status", "SweepPlan", "TraceRecord", "WoodburyBasis",
        "active_core", "cholesky_factor", "cholesky_solve", "column_partition",
        "compute_directions", "dot_tree", "duality_gap", "gen_random_feasible", "gram",
        "init_workspace", "mat_t_vec", "mat_vec", "parallel_sweep", "parse_problem",
        "prepare_woodbury", "rank_one_step", "scaled_gram", "scaling_diag", "serialize_problem",
        "solve_direct", "solve_lp", "solve_woodbury", "solve_woodbury_parallel", "step_length",
        "validate", "z_inverse_check"}
    assert set(P.__all__) == expected
    for name in expected:
        assert hasattr(P, name)


def test_solve_options_validation():
    P.SolveOptions()
    for bad in (dict(rho=0.0), dict(rho=1.0), dict(gap_tol=0.0), dict(max_iter=0),
                dict(backend="lu"), dict(workers=-1)):
        with pytest.raises(ValueError):
            P.SolveOptions(**bad)


def test_error_hierarchy():
    assert issubclass(P.SingularUpdate, ArithmeticError)
    assert issubclass(P.NotPositiveDefinite, ArithmeticError)
    for e in (P.DimensionMismatch, P.NonFiniteEntry, P.RankDeficient, P.NotInterior,
              P.NotFeasible, P.SchemaError):
        assert issubclass(e, ValueError) and issubclass(e, P.AdascaleError)
    assert issubclass(P.GenerationError, RuntimeError)


def test_dense_matrix_layout():
    A = P.DenseMatrix.from_rows([[1, 2, 3], [4, 5, 6]])
    assert list(A.data) == [1, 4, 2, 5, 3, 6]  # column-contiguous
    assert A.element(1, 2) == 6.0
    assert list(A.column(1)) == [2, 5]
    assert A.as_2d().flags.f_contiguous
    with pytest.raises(P.DimensionMismatch):
        P.DenseMatrix(2, 2, np.zeros(3))
    with pytest.raises(P.DimensionMismatch):
        A.column(3)


def test_lp_container_checks():
    A = P.DenseMatrix.from_rows([[1, 1]])
    P.StandardFormLP(A, [1.0], [1.0, 2.0])
    with pytest.raises(P.DimensionMismatch):
        P.StandardFormLP(A, [1.0, 2.0], [1.0, 2.0])
    with pytest.raises(P.DimensionMismatch):
        P.StandardFormLP(P.DenseMatrix.from_rows([[1], [1]]), [1.0, 1.0], [1.0])


def test_column_partition_semantics():
    plan = P.column_partition(10, 3, 1)  # live columns 0..10 (11) -> chunks of 4
    assert plan.assignments == {0: (0, 4), 1: (4, 8), 2: (8, 11)}
    assert plan.phase2_range(0, 1) == (1, 4)
    assert plan.active_columns() == set(range(11))
    plan = P.column_partition(4, 8, 4)  # 2 live columns, trailing workers idle
    assert plan.assignments[0] == (3, 4) and plan.assignments[7] == (5, 5)
    with pytest.raises(ValueError):
        P.column_partition(4, 0, 1)
    with pytest.raises(P.DimensionMismatch):
        P.column_partition(4, 2, 5)


def test_json_roundtrip_and_schema_errors():
    A = P.DenseMatrix.from_rows([[1, 1]])
    lp = P.StandardFormLP(A, [1.0], [1.0, 2.0])
    start = P.InteriorPoint([0.5, 0.5], [0.0], [1.0, 2.0])
    text = P.serialize_problem(lp, start)
    lp2, s2 = P.parse_problem(text)
    assert np.array_equal(lp2.A.data, lp.A.data) and np.array_equal(s2.s, start.s)
    for bad in ('[]', '{"m":1}', '{"m":1,"n":2,"A":[[1]],"b":[1],"c":[1,2]}',
                '{"m":true,"n":2,"A":[[1,1]],"b":[1],"c":[1,2]}', "{"):
        with pytest.raises(P.SchemaError):
            P.parse_problem(bad)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.NativeLibraryError):
        P.dot_tree([1.0, 2.0], [3.0, 4.0])
    lp = P.StandardFormLP(P.DenseMatrix.from_rows([[1, 1]]), [1.0], [1.0, 2.0])
    with pytest.raises(_lib.NativeLibraryError):
        P.solve_lp(lp, P.InteriorPoint([0.5, 0.5], [0.0], [1.0, 2.0]))


def test_active_core_names_cuda():
    assert P.active_core() == "cuda-sm_100a"


def test_harness_argument_parsing():
    from paper_1502_03543_b200 import harness as H

    assert H.parse_seed_range("1..4") == [1, 2, 3, 4] and H.parse_seed_range("7") == [7]
    for bad in ("4..1", "a..b", "x"):
        with pytest.raises(ValueError):
            H.parse_seed_range(bad)
    assert H.parse_grid("50x200,2000X20000") == [(50, 200), (2000, 20000)]
    with pytest.raises(ValueError):
        H.parse_grid("50by200")

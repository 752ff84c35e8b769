"""SPEC [OP] worked examples (reference SPEC.md, hand-derivable known answers)
expressed against the reference's kernel-table signatures, so the same cases
run against the CPU oracle (tests/test_oracle.py) and against the CUDA kernel
table (tests/test_gpu_kernels.py)."""

import math

import numpy as np


def F(rows):
    return np.asfortranarray(np.array(rows, dtype=np.float64))


def v(*xs):
    return np.array(xs, dtype=np.float64)


def chol(K, g):
    low, fail = K.cholesky_factor(F(g), 1e-12)
    return np.asarray(low), fail


def solve(K, low, b):
    return np.asarray(K.cholesky_solve_many(F(low), np.asarray(b, dtype=np.float64).reshape(-1, 1, order="F"))).ravel(order="F")


def case_dot_tree(K):
    # SPEC.md:45-47
    assert K.dot_tree(v(1, 2, 3, 4), v(1, 1, 1, 1)) == 10.0
    assert K.dot_tree(v(5), v(3)) == 15.0
    assert K.dot_tree(v(1, 2, 3), v(4, 5, 6)) == 32.0


def case_cholesky(K):
    # SPEC.md:54-56
    low, fail = chol(K, [[4, 2], [2, 3]])
    assert fail == -1
    assert np.array_equal(low, F([[2, 0], [1, math.sqrt(2.0)]]))
    low, fail = chol(K, np.eye(3))
    assert fail == -1 and np.array_equal(low, np.eye(3))
    _, fail = chol(K, [[1, 2], [2, 1]])
    assert fail == 1


def case_cholesky_solve(K):
    # SPEC.md:63-65
    assert np.array_equal(solve(K, np.eye(2), v(7, -3)), v(7, -3))
    low, _ = chol(K, [[4, 2], [2, 3]])
    assert np.allclose(solve(K, low, v(4, 3)), v(0.75, 0.5), rtol=0, atol=1e-15)
    assert np.array_equal(solve(K, np.diag([2.0, 3.0]), v(8, 18)), v(2, 2))


def case_gram(K):
    # SPEC.md:72-74, 81-83
    assert np.array_equal(np.asarray(K.gram(F([[1, 0, 0], [0, 1, 0]]))), np.eye(2))
    assert np.array_equal(np.asarray(K.gram(F([[1, 1]]))), F([[2]]))
    assert np.array_equal(np.asarray(K.gram(F([[1, 2], [3, 4]]))), F([[5, 11], [11, 25]]))
    assert np.array_equal(np.asarray(K.scaled_gram(F([[1, 1]]), v(0.5, 0.25))), F([[0.75]]))
    a = F([[1, 2, 3], [4, 5, 6]])
    assert np.array_equal(np.asarray(K.scaled_gram(a, v(1, 1, 1))), np.asarray(K.gram(a)))
    assert np.array_equal(np.asarray(K.scaled_gram(np.asfortranarray(np.eye(2)), v(2, 5))), np.diag([2.0, 5.0]))


def case_mat_vec(K):
    # SPEC.md:90-92
    assert np.array_equal(np.asarray(K.mat_vec(F([[1, 1]]), v(0.5, 0.5))), v(1.0))
    assert np.array_equal(np.asarray(K.mat_t_vec(F([[1, 1]]), v(4 / 3))), v(4 / 3, 4 / 3))
    x = v(0.3, -2.5, 7.25)
    assert np.array_equal(np.asarray(K.mat_vec(np.asfortranarray(np.eye(3)), x)), x)


def case_cascade(K):
    # SPEC.md:223-225 (prepare), 232-234 (init), 243 (rank_one_step), 254
    a = F([[2]])
    low, fail = chol(K, np.asarray(K.gram(a)))
    assert fail == -1 and low[0, 0] == 2.0
    y = np.asarray(K.cholesky_solve_many(F(low), a))
    assert y[0, 0] == 0.5
    x0 = solve(K, low, v(6))
    assert x0[0] == 1.5
    cols = F([[0.5, 1.5]])
    inner = np.zeros(2)
    vv = np.zeros(1)
    K.build_v(a, 0, 3.0, vv)
    assert vv[0] == 4.0
    K.sweep_phase1(cols, vv, inner, 0, 2)
    assert list(inner) == [2.0, 6.0]
    K.sweep_phase2(cols, 0, inner, 1.0 + inner[0], 1, 2)
    assert cols[0, 1] == 0.5
    # full cascade, same system
    cols = F([[0.5, 1.5]])
    assert K.solve_sweeps(cols, a, v(3.0), np.zeros(2), np.zeros(1), 1) == 0
    assert cols[0, 1] == 0.5
    # identity A, d=(2,5), b=(4,10) -> (2,2)
    a = np.asfortranarray(np.eye(2))
    cols = F([[1, 0, 4], [0, 1, 10]])
    assert K.solve_sweeps(cols, a, v(2, 5), np.zeros(3), np.zeros(2), 1) == 0
    assert np.array_equal(cols[:, 2], v(2, 2))
    # d = 0 on A=[[1]]: denom = 1 + (-1)(1) = 0 -> breakdown at step 1
    cols = F([[1.0, 1.0]])
    assert K.solve_sweeps(cols, F([[1]]), v(0.0), np.zeros(2), np.zeros(1), 1) == 1


CASES = [case_dot_tree, case_cholesky, case_cholesky_solve, case_gram, case_mat_vec, case_cascade]

# Worked LP: A=[[1,1]], b=1, c=(1,2), x=(.5,.5), y=0, s=(1,2)
WORKED = dict(A=F([[1, 1]]), b=v(1), c=v(1, 2), x=v(0.5, 0.5), y=v(0.0), s=v(1, 2))
WORKED_DY = 4 / 3
WORKED_ALPHA1 = 0.675
# reference compiled core (run here): gap_tol=1e-6 -> 8 iterations, c'x =
# 1.0000008818438226; default gap_tol -> 10 iterations, c'x = 1.0000000035096694
WORKED_RUNS = [(1e-6, 8, 1.0000008818438226), (None, 10, 1.0000000035096694)]

"""Restatement of proj/tests/test_driver.cpp / test_sketch.cpp / test_pinv.cpp essentials
against the oracle (same mt19937_64 fixtures where the reference uses them)."""
import math

import numpy as np
import pytest


def test_sketch_rows_for_block(oracle):  # test_sketch.cpp:20-32
    assert [oracle.sketch_rows_for_block(b) for b in (1, 10, 50, 100, 250)] == [1, 11, 55, 110, 275]


def test_identity_input_copies_embedding(oracle):
    y, _, _ = oracle.sketch(np.eye(4), 2, 9)
    assert y.shape == (2, 4)
    assert np.array_equal(y, oracle.gaussian_matrix(2, 4, 9, 1))


def test_same_seed_bitwise_identical_sketch(oracle):  # test_sketch.cpp:34-42
    a = oracle.random_dense(12, 10, 2)
    y1, _, _ = oracle.sketch(a, 3, 42)
    y2, _, _ = oracle.sketch(a, 3, 42)
    y3, _, _ = oracle.sketch(a, 3, 43)
    assert np.array_equal(y1, y2) and not np.array_equal(y1, y3)


def test_sketch_validation(oracle):  # test_sketch.cpp:54-59
    a = oracle.random_dense(4, 6, 1)
    with pytest.raises(ValueError):
        oracle.sketch(a, 0, 0)
    with pytest.raises(ValueError, match="block exceeds row count"):
        oracle.sketch(a, 5, 0)


def test_adjusted_threshold_4_98(oracle):  # test_driver.cpp:27-32
    xi = oracle.adjusted_threshold(1.0, 0.0, 1e-10, 100)
    assert xi == pytest.approx(1 / 4.98, rel=5e-4)
    assert oracle.adjusted_threshold(1e-6, 0.0, 1e-10, 100) == pytest.approx(xi * 1e-6, rel=1e-12)


def test_adjusted_threshold_closed_form_and_boundary(oracle):  # 34-58
    c, alpha, delta, eps = 110.0, 0.01, 1.0, 1e-4
    want = (1 + delta) * math.sqrt(1 - 2 * math.sqrt(-math.log(alpha) / c)) * eps
    assert oracle.adjusted_threshold(eps, delta, alpha, 110) == pytest.approx(want, rel=1e-15)
    ba = math.exp(-100 / 4.0)
    with pytest.raises(ValueError, match="block too small"):
        oracle.adjusted_threshold(1.0, 0.0, ba, 100)
    nearly = oracle.adjusted_threshold(1.0, 0.0, ba * 1.001, 100)
    assert 0 < nearly < 0.05
    with pytest.raises(ValueError):
        oracle.adjusted_threshold(1e-3, 0.0, 1.5, 100)
    with pytest.raises(ValueError):
        oracle.adjusted_threshold(1e-3, -0.5, 0.1, 100)


def test_gratton_tail(oracle):  # 60-66
    assert oracle.gratton_tail(4, math.sqrt(2)) == pytest.approx(math.exp(-0.25), rel=1e-12)
    assert oracle.gratton_tail(100, 2.0) == pytest.approx(math.exp(-900 / 64), rel=1e-12)
    with pytest.raises(ValueError):
        oracle.gratton_tail(50, 1.0)
    with pytest.raises(ValueError):
        oracle.gratton_tail(0, 2.0)


def test_rank1_one_iteration(oracle):  # 68-81
    a = oracle.random_gaussian(100, 1, 5) @ oracle.random_gaussian(80, 1, 6).T
    r = oracle.iterative_cur(a, epsilon=1e-8, b=5, seed=3)
    assert r.status == "Converged" and len(r.rhos) == 1 and r.rank <= 5
    assert oracle.true_relative_error(a, r.row_indices, r.col_indices) <= 1e-10


def test_exact_rank20_in_two_blocks(oracle):  # 83-96
    a = oracle.random_gaussian(300, 20, 7) @ oracle.random_gaussian(250, 20, 8).T
    r = oracle.iterative_cur(a, epsilon=1e-6, b=10, seed=11)
    assert r.status == "Converged" and r.rank == 20 and len(r.rhos) == 2
    assert oracle.true_relative_error(a, r.row_indices, r.col_indices) <= 1e-10


def test_block_too_small_for_alpha(oracle):  # 121-130
    a = oracle.random_dense(40, 40, 23)
    with pytest.raises(ValueError, match="block too small"):
        oracle.iterative_cur(a, epsilon=1e-4, b=2, alpha=0.1, risk_adjust=True, seed=1)


def test_epsilon_at_or_above_one(oracle):  # 132-143
    r = oracle.iterative_cur(oracle.random_dense(10, 10, 29), epsilon=1.0, b=2, seed=0)
    assert r.status == "Converged" and r.rank == 0 and r.final_rho == 1.0 and r.note


def test_zero_matrix_rejected(oracle):  # 145-149
    with pytest.raises(ValueError, match="nonzero"):
        oracle.iterative_cur(np.zeros((5, 5)))


def test_fixed_rank_stops_exactly(oracle):  # 151-160
    r = oracle.iterative_cur(oracle.random_dense(50, 45, 31), epsilon=0.0, b=7, max_rank=23, seed=2)
    assert r.status == "MaxRank" and r.rank == 23


def test_exact_interpolation_2x2(oracle):  # 192-207
    a = np.array([[1.0, 0.0], [0.0, 0.0]])
    r = oracle.iterative_cur(a, epsilon=0.0, b=1, max_rank=2, seed=3)
    assert r.status == "Converged" and r.final_rho == 0.0 and r.rank == 1


def test_true_error_basics_and_core(oracle):  # 227-238, test_pinv make_cur_factors exactness
    a = oracle.random_dense(10, 8, 43)
    assert oracle.true_relative_error(a, [], []) == 1.0
    sq = oracle.random_dense(8, 8, 44)
    idx = list(range(8))
    assert oracle.true_relative_error(sq, idx, idx) <= 1e-13
    core = oracle.core_matrix(sq, idx, idx)
    assert np.allclose(core @ sq, np.eye(8), atol=1e-10)


def test_recurrence_identity(oracle):  # test_driver.cpp:259-283 residual recurrence (restated numerically)
    for seed in range(10):
        a = oracle.random_gaussian(12, 12, 700 + seed)
        i0, j0, i1, j1 = [0, 3], [1, 5], [7, 9], [2, 8]

        def resid(x, I, J):
            return x - x[:, J] @ np.linalg.solve(x[np.ix_(I, J)], x[I, :])

        s = resid(a, i0, j0)
        lhs_small = resid(s, i1, j1)
        lhs_full = resid(a, i0 + i1, j0 + j1)
        assert np.linalg.norm(lhs_full - lhs_small) <= 1e-9 * np.linalg.norm(a)


def test_sparse_sign_run_converges(oracle):
    a = oracle.random_gaussian(120, 10, 3) @ oracle.random_gaussian(90, 10, 4).T
    r = oracle.iterative_cur(a, epsilon=1e-8, b=5, seed=7, sketch="sparse_sign")
    assert r.status == "Converged" and r.rank == 10
    assert oracle.true_relative_error(a, r.row_indices, r.col_indices) <= 1e-10


def test_oracle_slupp_exact_rank(oracle):  # proj/tests/test_baselines.cpp:53-57
    a = oracle.random_gaussian(60, 7, 11) @ oracle.random_gaussian(50, 7, 12).T
    I, J = oracle.slupp_cur(a, 7, 13)
    assert len(I) == 7 and len(J) == 7
    assert oracle.true_relative_error(a, I, J) <= 1e-10
    with pytest.raises(Exception, match="rank must lie"):
        oracle.slupp_cur(a, 51, 0)

"""Restatement of proj/tests/test_select.cpp against the oracle (same mt19937_64 fixtures)."""
import numpy as np
import pytest


def lupp_reference_pivots(w, steps):
    """proj/tests/oracles.hpp:100-119: row-swapping Gaussian elimination with partial pivoting."""
    w = np.array(w, dtype=np.float64)
    original = list(range(w.shape[0]))
    pivots = []
    for s in range(min(steps, w.shape[0], w.shape[1])):
        best = s
        for i in range(s, w.shape[0]):
            if abs(w[i, s]) > abs(w[best, s]):
                best = i
        if w[best, s] == 0.0:
            break
        w[[s, best]] = w[[best, s]]
        original[s], original[best] = original[best], original[s]
        pivots.append(original[s])
        for i in range(s + 1, w.shape[0]):
            f = w[i, s] / w[s, s]
            w[i, s:] -= f * w[s, s:]
    return pivots


def test_first_lupp_column_pivot(oracle):  # test_select.cpp:25-30
    m = np.array([[1.0, 0, 3], [0, 2, 0]])
    got = oracle.select_columns(m, 1)
    assert got.indices == [2] and got.last_pivot_magnitude == 3.0


def test_lupp_matches_row_swapping_elimination(oracle):  # test_select.cpp:52-60
    m = oracle.random_dense(50, 5, 13)
    assert oracle.select_rows(m, 5).indices == lupp_reference_pivots(m, 5)
    wide = oracle.random_dense(80, 8, 14)
    assert oracle.select_columns(wide.T, 6).indices == lupp_reference_pivots(wide, 6)


def test_single_column_row_selection(oracle):  # 62-68
    assert oracle.select_rows(np.array([[0.0], [5.0], [1.0]]), 1).indices == [1]


def test_masked_rows_never_selected(oracle):  # 70-79
    m = oracle.random_dense(10, 4, 17)
    m[:4, :] = 0.0
    got = oracle.select_rows(m, 2, exclude=[0, 1, 2, 3])
    assert len(got.indices) == 2 and all(i >= 4 for i in got.indices)


def test_selection_is_deterministic(oracle):  # 81-91
    m = oracle.random_dense(15, 40, 23)
    a = oracle.select_columns(m, 6, exclude=[3, 9])
    b = oracle.select_columns(m, 6, exclude=[3, 9])
    assert a == b


def test_indices_distinct_and_avoid_exclusions(oracle):  # 93-106
    for seed in range(10):
        m = oracle.random_dense(12, 30, 400 + seed)
        ex = [0, 5, 11, 17, 29]
        got = oracle.select_columns(m, 8, exclude=ex)
        assert len(set(got.indices)) == len(got.indices)
        assert not set(got.indices) & set(ex)


def test_permutation_equivariance(oracle):  # 108-125
    m = oracle.random_dense(10, 25, 57)
    perm = np.random.default_rng(3).permutation(25)
    permuted = np.empty_like(m)
    permuted[:, perm] = m
    base = oracle.select_columns(m, 6)
    moved = oracle.select_columns(permuted, 6)
    assert moved.indices == [int(perm[i]) for i in base.indices]


def test_truncation_on_exhausted_residual(oracle):  # 127-142
    m = oracle.random_gaussian(8, 2, 61) @ oracle.random_gaussian(30, 2, 62).T
    got = oracle.select_columns(m, 5)
    assert got.truncated and len(got.indices) == 2
    empty = oracle.select_columns(np.zeros((6, 9)), 3)
    assert empty.indices == [] and empty.truncated


def test_row_selection_caps_at_width(oracle):  # 144-149
    got = oracle.select_rows(oracle.random_dense(20, 3, 67), 5)
    assert len(got.indices) == 3 and got.truncated


def test_validation(oracle):  # 151-161
    m = oracle.random_dense(4, 9, 71)
    with pytest.raises(ValueError):
        oracle.select_columns(m, 5)
    with pytest.raises(ValueError):
        oracle.select_columns(m, 2, pivot_floor=0.0)
    with pytest.raises(IndexError):
        oracle.select_columns(m, 2, exclude=[40])
    with pytest.raises(RuntimeError, match="not implemented"):
        oracle.select_columns(m, 2, method="osinsky")
    with pytest.raises(RuntimeError, match="not implemented"):
        oracle.select_rows(m, 2, method="osinsky")


def test_dependent_selection_example(oracle):  # 163-194
    n, eta = 100, 1e-3
    a = np.zeros((2, n + 1))
    a[0, 1:] = 1.0 / np.sqrt(n)
    a[1, 0] = 1.0 / np.sqrt(n) + eta
    col = oracle.select_columns(a, 1, method="qrcp")
    assert col.indices == [0]
    row = oracle.select_rows(a[:, [0]], 1)
    assert row.indices == [1]
    assert a[row.indices[0], col.indices[0]] != 0.0

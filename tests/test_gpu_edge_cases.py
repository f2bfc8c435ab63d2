"""Edge cases of the IterativeCUR path on the B200 against the CPU oracle: degenerate and extreme
shapes, a block as large as the matrix, exact ties in the pivot searches (the reference breaks them
toward the lowest index, select.cpp:34-74), zero rows/columns, budgets of one, runs to exhaustion,
risk-adjusted stopping, a padded leading dimension, and both sketches."""
import numpy as np
import pytest

from parity_util import compare_runs

pytestmark = pytest.mark.gpu


def check(engine, oracle, a, **kw):
    f, t = engine.iterative_cur(a, **kw)
    o = oracle.iterative_cur(a, **kw)
    v = compare_runs(o, f, t)
    assert v["status_equal"], (t.status, o.status, kw)
    assert v["identical"], (v, kw)
    err = engine.true_relative_error(a, f)
    err_o = oracle.true_relative_error(a, o.row_indices, o.col_indices)
    assert abs(err - err_o) <= 1e-8, (err, err_o, kw)
    return f, t, o


@pytest.mark.parametrize("shape,b", [((1, 1), 1), ((1, 7), 1), ((9, 1), 1), ((3, 200), 2), ((20000, 3), 3),
                                     ((40, 40), 40), ((37, 23), 23), ((64, 5), 5)])
@pytest.mark.parametrize("sketch", ["gaussian", "sparse_sign"])
def test_extreme_shapes(engine, oracle, shape, b, sketch):
    if sketch == "sparse_sign" and (b * 11) // 10 < 1:
        pytest.skip("no sketch rows")
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    m, n = shape
    r = min(m, n, 4)
    a = rng.standard_normal((m, r)) @ rng.standard_normal((r, n)) + 1e-3 * rng.standard_normal((m, n))
    check(engine, oracle, a, epsilon=1e-8, b=b, seed=3, sketch=sketch)


def test_block_equal_to_the_row_count(engine, oracle):
    rng = np.random.default_rng(2)
    a = rng.standard_normal((30, 50))
    f, t, o = check(engine, oracle, a, epsilon=1e-12, b=30, seed=1)
    assert f.rank == o.rank


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_exact_ties_break_to_the_lowest_index(engine, oracle, seed):
    """Duplicated columns and rows: the pivot searches meet exactly equal magnitudes."""
    rng = np.random.default_rng(seed)
    base = rng.integers(-3, 4, size=(60, 8)).astype(np.float64)
    a = np.concatenate([base, base, base[:, ::-1]], axis=1)          # 24 columns, 3 copies
    a = np.concatenate([a, a[:20]], axis=0)                          # 80 rows, 20 duplicated
    check(engine, oracle, a, epsilon=1e-10, b=4, seed=seed)
    check(engine, oracle, a, epsilon=1e-10, b=4, seed=seed, sketch="sparse_sign")


def test_integer_matrix_with_many_equal_magnitudes(engine, oracle):
    rng = np.random.default_rng(7)
    a = rng.choice([-1.0, 0.0, 1.0], size=(120, 90))
    check(engine, oracle, a, epsilon=1e-6, b=6, seed=2)


def test_zero_rows_and_columns(engine, oracle):
    rng = np.random.default_rng(4)
    a = rng.standard_normal((70, 6)) @ rng.standard_normal((6, 50))
    a[::7, :] = 0.0
    a[:, ::5] = 0.0
    f, t, o = check(engine, oracle, a, epsilon=1e-10, b=4, seed=5)
    assert all(j % 5 for j in f.col_indices) and all(i % 7 for i in f.row_indices)


@pytest.mark.parametrize("kw", [dict(max_iters=1), dict(max_rank=1), dict(max_rank=7, b=3), dict(max_iters=2, b=1)])
def test_budgets_of_one(engine, oracle, kw):
    rng = np.random.default_rng(8)
    a = rng.standard_normal((80, 60))
    base = dict(epsilon=1e-12, b=5, seed=1)
    base.update(kw)
    f, t, o = check(engine, oracle, a, **base)
    assert t.status == "MaxRank"


def test_run_to_exhaustion_on_exact_low_rank(engine, oracle):
    """epsilon = 0 on an exact rank-6 product: the floors end the run (ResidualExhausted or the
    rank budget), exactly where the oracle's do."""
    a = oracle.random_gaussian(90, 6, 21) @ oracle.random_gaussian(70, 6, 22).T
    f, t, o = check(engine, oracle, a, epsilon=0.0, b=4, seed=2)
    assert f.rank >= 6


def test_risk_adjusted_run(engine, oracle):
    rng = np.random.default_rng(9)
    u, _ = np.linalg.qr(rng.standard_normal((300, 200)))
    v, _ = np.linalg.qr(rng.standard_normal((200, 200)))
    a = (u * 0.9 ** np.arange(200)) @ v.T
    f, t, o = check(engine, oracle, a, epsilon=1e-5, b=25, seed=3, risk_adjust=True, delta=0.1, alpha=0.05)
    assert t.threshold == pytest.approx(o.threshold, rel=1e-15)


def test_sparse_sign_every_row_hit(engine, oracle):
    """b = 8: c = floor(1.1 * 8) = 8 = zeta, so every sketch row receives every row of A."""
    rng = np.random.default_rng(10)
    a = rng.standard_normal((200, 12)) @ rng.standard_normal((12, 150))
    check(engine, oracle, a, epsilon=1e-9, b=8, seed=4, sketch="sparse_sign")


def test_padded_leading_dimension_device_entry(engine, oracle):
    import torch

    rng = np.random.default_rng(11)
    a = rng.standard_normal((333, 20)) @ rng.standard_normal((20, 211))
    buf = torch.zeros(211, 350, dtype=torch.float64, device="cuda")  # ld 350 > m = 333
    buf[:, :333] = torch.from_numpy(np.ascontiguousarray(a.T))
    t = buf.t()[:333, :]
    assert t.stride() == (1, 350)
    f, tr = engine.iterative_cur(engine.MatrixHandle.device(t), epsilon=1e-10, b=7, seed=2)
    o = oracle.iterative_cur(a, epsilon=1e-10, b=7, seed=2)
    v = compare_runs(o, f, tr)
    assert v["status_equal"] and v["identical"], v
    assert abs(engine.true_relative_error(engine.MatrixHandle.device(t), f) -
               oracle.true_relative_error(a, o.row_indices, o.col_indices)) <= 1e-8

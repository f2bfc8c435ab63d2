"""GPU parity of the full IterativeCUR path (public API -> C-ABI -> sm_100a kernels) against
the CPU oracle, plus the reference's own driver / smoke tests restated through the engine."""
import math

import numpy as np
import pytest

from parity_util import compare_runs

pytestmark = pytest.mark.gpu


def exp_decay(n, ratio, seed_rng):
    q1, _ = np.linalg.qr(seed_rng.standard_normal((n, n)))
    q2, _ = np.linalg.qr(seed_rng.standard_normal((n, n)))
    return (q1 * ratio ** np.arange(n)) @ q2.T


def low_rank_plus_noise(oracle, m, n, r, rel_noise, seed):
    a = oracle.random_gaussian(m, r, seed) @ oracle.random_gaussian(n, r, seed + 1).T
    noise = oracle.random_gaussian(m, n, seed + 2)
    return a + (rel_noise * np.linalg.norm(a) / np.linalg.norm(noise)) * noise


@pytest.mark.parametrize("case", ["expdecay600", "lowrank_noise", "rbf1500", "sparse_sign", "sparse_sign_b40",
                                  "sparse_sign_b40_tcgen05", "sparse_sign_b40_mma_s8", "sparse_sign_b40_dmma",
                                  "sparse_sign_b50_tall", "odd_shape", "b64", "b1"])
def test_engine_matches_oracle(engine, oracle, case):
    rng = np.random.default_rng(11)
    kw = dict(epsilon=1e-6, b=10, seed=0)
    if case == "expdecay600":
        a = exp_decay(600, 10 ** (-1 / 20), rng)
    elif case == "lowrank_noise":
        a = low_rank_plus_noise(oracle, 500, 400, 60, 1e-9, 5)
        kw.update(epsilon=1e-7, b=16, seed=3)
    elif case == "rbf1500":
        x, y = rng.random((1500, 3)), rng.random((1200, 3))
        d2 = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
        a = np.exp(-d2 / (2 * 0.5 ** 2))
        kw.update(epsilon=1e-8, b=32, seed=1)
    elif case == "sparse_sign":
        u, _ = np.linalg.qr(rng.standard_normal((800, 400)))
        v, _ = np.linalg.qr(rng.standard_normal((400, 400)))
        a = (u * (np.arange(1, 401) ** -2.0)) @ v.T
        kw.update(epsilon=1e-4, b=20, seed=2, sketch="sparse_sign")
    elif case.startswith("sparse_sign_b40"):  # c_pad = 48 through each sparse-sign sketch kernel
        import os

        mode = {"sparse_sign_b40": "1", "sparse_sign_b40_tcgen05": "", "sparse_sign_b40_mma_s8": "2",
                "sparse_sign_b40_dmma": "0"}[case]  # "" = the default (tcgen05 above c_pad 32)
        if mode:
            os.environ["ITERCUR_SPARSE_SKETCH"] = mode
        a = low_rank_plus_noise(oracle, 900, 700, 120, 1e-9, 13)
        kw.update(epsilon=1e-7, b=40, seed=5, sketch="sparse_sign")
    elif case == "sparse_sign_b50_tall":  # config 4's block size (c = 55), tcgen05 sketch, split K
        a = low_rank_plus_noise(oracle, 6000, 900, 140, 1e-10, 17)
        kw.update(epsilon=1e-8, b=50, seed=7, sketch="sparse_sign")
    elif case == "b64":  # wide blocks: block-level LU and 64-wide solves (configs 4/5 use b = 50 / 64)
        a = low_rank_plus_noise(oracle, 700, 520, 150, 1e-10, 21)
        kw.update(epsilon=1e-8, b=64, seed=6)
    elif case == "b1":  # c = 1 sketch row, one pivot per block
        a = low_rank_plus_noise(oracle, 90, 70, 6, 1e-12, 31)
        kw.update(epsilon=1e-9, b=1, seed=8)
    else:
        a = low_rank_plus_noise(oracle, 333, 217, 25, 1e-11, 9)
        kw.update(epsilon=1e-9, b=7, seed=4)
    try:
        f, t = engine.iterative_cur(a, **kw)
    finally:
        import os

        os.environ.pop("ITERCUR_SPARSE_SKETCH", None)
    o = oracle.iterative_cur(a, **kw)
    v = compare_runs(o, f, t)
    assert v["status_equal"], (o.status, t.status)
    assert v["identical"], v
    err = engine.true_relative_error(a, f)
    err_o = oracle.true_relative_error(a, o.row_indices, o.col_indices)
    assert abs(err - err_o) <= 1e-8, (err, err_o)
    if v["full_identical"]:
        assert len(t.rhos) == len(o.rhos)
        # late rho values are cancellation-limited: compare on the scale of rho_0 = 1
        assert np.allclose(t.rhos, o.rhos, rtol=1e-6, atol=1e-9)
    # the device-evaluated error agrees with the oracle's for the engine's own indices
    err_e_o = oracle.true_relative_error(a, f.row_indices, f.col_indices)
    assert abs(err - err_e_o) <= 1e-9 + 0.1 * err_e_o


def test_config1_full_size_matches_oracle(engine, oracle):
    """BASELINE config 1 at full size: 2000 x 2000, sigma_i = 10^(-(i-1)/20), b = 10, tol 1e-6."""
    rng = np.random.default_rng(1)
    a = exp_decay(2000, 10 ** (-1 / 20), rng)
    kw = dict(epsilon=1e-6, b=10, seed=0)
    f, t = engine.iterative_cur(a, **kw)
    o = oracle.iterative_cur(a, **kw)
    v = compare_runs(o, f, t)
    assert v["status_equal"] and v["identical"], v
    err = engine.true_relative_error(a, f)
    err_o = oracle.true_relative_error(a, o.row_indices, o.col_indices)
    assert abs(err - err_o) <= 1e-8


# ------------------------- proj/tests/test_driver.cpp restated through the engine --------
def test_rank1_converges_in_one_iteration(engine, oracle):
    a = oracle.random_gaussian(100, 1, 5) @ oracle.random_gaussian(80, 1, 6).T
    f, t = engine.iterative_cur(a, epsilon=1e-8, b=5, seed=3)
    assert t.status == "Converged" and len(t.iterations) == 1 and f.rank <= 5
    assert engine.true_relative_error(a, f) <= 1e-10


def test_exact_rank20_two_blocks_of_10(engine, oracle):
    a = oracle.random_gaussian(300, 20, 7) @ oracle.random_gaussian(250, 20, 8).T
    f, t = engine.iterative_cur(a, epsilon=1e-6, b=10, seed=11)
    assert t.status == "Converged" and f.rank == 20 and len(t.iterations) == 2
    assert engine.true_relative_error(a, f) <= 1e-10


def test_risk_adjust_block_too_small(engine, oracle):
    with pytest.raises(ValueError, match="block too small"):
        engine.iterative_cur(oracle.random_dense(40, 40, 23), epsilon=1e-4, b=2, alpha=0.1, risk_adjust=True, seed=1)


def test_epsilon_at_or_above_one(engine, oracle):
    f, t = engine.iterative_cur(oracle.random_dense(10, 10, 29), epsilon=1.0, b=2, seed=0)
    assert t.status == "Converged" and f.rank == 0 and t.final_rho == 1.0 and t.note
    assert engine.true_relative_error(oracle.random_dense(10, 10, 29), f) == 1.0


def test_zero_matrix_rejected(engine):
    with pytest.raises(ValueError):
        engine.iterative_cur(np.zeros((4, 4)), epsilon=1e-3, b=2)  # test_smoke.py:81-84
    with pytest.raises(ValueError, match="nonzero"):
        engine.iterative_cur(np.zeros((5, 5)))


def test_validation_messages(engine, oracle):
    a = oracle.random_dense(4, 6, 1)
    with pytest.raises(ValueError, match="block exceeds row count"):
        engine.iterative_cur(a, b=5)
    with pytest.raises(ValueError, match="block size"):
        engine.iterative_cur(a, b=0)
    with pytest.raises(ValueError, match="epsilon"):
        engine.iterative_cur(a, epsilon=-1.0, b=2)
    with pytest.raises(ValueError, match="non-finite"):
        bad = a.copy()
        bad[1, 1] = np.nan
        engine.iterative_cur(bad, b=2)
    with pytest.raises(RuntimeError, match="not implemented"):
        engine.iterative_cur(oracle.random_dense(20, 20, 3), b=2, col_method="osinsky")
    with pytest.raises(ValueError, match="unknown selection method"):
        engine.iterative_cur(a, b=2, col_method="bogus")


def test_fixed_rank_stops_at_max_rank(engine, oracle):
    f, t = engine.iterative_cur(oracle.random_dense(50, 45, 31), epsilon=0.0, b=7, max_rank=23, seed=2)
    assert t.status == "MaxRank" and f.rank == 23


def test_rank_grows_by_recorded_blocks(engine, oracle):
    a = low_rank_plus_noise(oracle, 60, 50, 12, 1e-4, 37)
    f, t = engine.iterative_cur(a, epsilon=1e-3, b=5, seed=4)
    assert sum(r.cols_added for r in t.iterations) == f.rank == len(f.row_indices)
    assert all(r.cols_added == r.rows_added >= 1 for r in t.iterations)


def test_iteration_budget(engine, oracle):
    for seed in range(3):
        a = low_rank_plus_noise(oracle, 40, 30, 6, 1e-2, 600 + seed)
        _, t = engine.iterative_cur(a, epsilon=1e-8, b=4, seed=seed)
        assert len(t.iterations) <= (30 + 3) // 4 + 1


def test_exact_interpolation_2x2(engine):
    a = np.array([[1.0, 0.0], [0.0, 0.0]])
    f, t = engine.iterative_cur(a, epsilon=0.0, b=1, max_rank=2, seed=3)
    assert t.status == "Converged" and t.final_rho == 0.0 and f.rank == 1
    assert engine.true_relative_error(a, f) <= 1e-14


def test_past_numerical_rank(engine, oracle):
    a = oracle.random_gaussian(30, 3, 41) @ oracle.random_gaussian(25, 3, 42).T
    f, t = engine.iterative_cur(a, epsilon=0.0, b=3, max_rank=10, seed=5)
    assert 3 <= f.rank <= 10
    assert engine.true_relative_error(a, f) <= 1e-10


def test_factors_reconstruct_the_matrix(engine, oracle):  # test_smoke.py:46-52
    a = oracle.random_gaussian(40, 5, 1) @ oracle.random_gaussian(30, 5, 2).T
    f, _ = engine.iterative_cur(a, epsilon=1e-8, b=5, seed=2)
    approx = f.c_matrix() @ f.core_matrix() @ f.r_matrix()
    assert np.linalg.norm(a - approx) / np.linalg.norm(a) <= 1e-9
    assert np.array_equal(f.c_matrix(), a[:, f.col_indices])
    assert np.array_equal(f.r_matrix(), a[f.row_indices, :])
    core_o = oracle.core_matrix(a, f.row_indices, f.col_indices)
    assert np.allclose(f.core_matrix(), core_o, rtol=1e-8, atol=1e-10 * np.abs(core_o).max())


def test_core_matrix_multi_block(engine, oracle):
    a = low_rank_plus_noise(oracle, 200, 150, 30, 1e-6, 71)
    f, t = engine.iterative_cur(a, epsilon=1e-9, b=8, seed=1)
    assert len(t.iterations) >= 3
    core = f.core_matrix()
    X = a[np.ix_(f.row_indices, f.col_indices)]
    assert np.linalg.norm(core @ X - np.eye(f.rank)) <= 1e-8 * np.linalg.cond(X)


def test_sketched_estimate_tracks_truth(engine, oracle):  # test_driver.cpp:307-320 (20 draws)
    in_band = 0
    for seed in range(20):
        a = low_rank_plus_noise(oracle, 150, 150, 10, 1e-5, 1000 + seed * 3)
        f, t = engine.iterative_cur(a, epsilon=1e-4, b=50, seed=seed)
        truth = engine.true_relative_error(a, f)
        if 0.5 <= t.final_rho / truth <= 2.0:
            in_band += 1
    assert in_band >= 18


def test_device_entry_with_torch_tensor(engine, oracle):
    import torch

    a = oracle.random_gaussian(300, 20, 7) @ oracle.random_gaussian(250, 20, 8).T
    t_a = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()  # column-major view
    f, t = engine.iterative_cur(engine.MatrixHandle.device(t_a), epsilon=1e-6, b=10, seed=11)
    f2, t2 = engine.iterative_cur(a, epsilon=1e-6, b=10, seed=11)
    assert f.row_indices == f2.row_indices and f.col_indices == f2.col_indices
    assert t.rhos == t2.rhos  # deterministic run to run


def test_closed_forms(engine):  # test_smoke.py:65-69
    assert engine.adjusted_threshold(1.0, 0.0, 1e-10, 100) == pytest.approx(1 / 4.98, rel=5e-4)
    assert engine.gratton_tail(4, math.sqrt(2.0)) == pytest.approx(math.exp(-0.25))


# ------------------------- s-LUPP one-shot baseline (proj/src/baselines.cpp:39-62) ---------
def test_slupp_recovers_exact_rank(engine, oracle):  # proj/tests/test_baselines.cpp:53-57
    a = oracle.random_gaussian(60, 7, 11) @ oracle.random_gaussian(50, 7, 12).T
    f = engine.slupp_cur(a, 7, 13)
    assert f.rank == 7
    assert engine.true_relative_error(a, f) <= 1e-10


@pytest.mark.parametrize("rank,seed", [(10, 0), (25, 3), (64, 1)])
def test_slupp_matches_oracle(engine, oracle, rank, seed):
    rng = np.random.default_rng(rank)
    a = exp_decay(300, 10 ** (-1 / 30), rng)[:, :240]
    f = engine.slupp_cur(a, rank, seed)
    I, J = oracle.slupp_cur(a, rank, seed)
    assert f.row_indices == I and f.col_indices == J
    err = engine.true_relative_error(a, f)
    assert abs(err - oracle.true_relative_error(a, I, J)) <= 1e-8


def test_slupp_validation(engine, oracle):
    a = oracle.random_dense(10, 8, 3)
    with pytest.raises(ValueError, match="rank must lie"):
        engine.slupp_cur(a, 9)
    assert engine.slupp_cur(a, 0).rank == 0


@pytest.mark.parametrize("cm,rm", [("qrcp", "qrcp"), ("qrcp", "lupp"), ("lupp", "qrcp")])
def test_qrcp_methods_match_oracle(engine, oracle, cm, rm):
    a = low_rank_plus_noise(oracle, 260, 200, 30, 1e-10, 51)
    kw = dict(epsilon=1e-8, b=8, seed=3, col_method=cm, row_method=rm)
    f, t = engine.iterative_cur(a, **kw)
    o = oracle.iterative_cur(a, **kw)
    assert t.status == o.status
    assert f.row_indices == list(o.row_indices) and f.col_indices == list(o.col_indices)
    err = engine.true_relative_error(a, f)
    assert abs(err - oracle.true_relative_error(a, o.row_indices, o.col_indices)) <= 1e-8


def test_sparse_csr_input_matches_dense(engine, oracle):  # MatrixHandle.sparse_csr path
    a = low_rank_plus_noise(oracle, 120, 90, 8, 1e-10, 61)
    a[np.abs(a) < 0.5 * np.abs(a).mean()] = 0.0
    rows, cols = np.nonzero(a)
    indptr = np.searchsorted(rows, np.arange(a.shape[0] + 1))
    h = engine.MatrixHandle.sparse_csr(a.shape[0], a.shape[1], indptr, cols, a[rows, cols])
    f, t = engine.iterative_cur(h, epsilon=1e-6, b=5, seed=1)
    f2, t2 = engine.iterative_cur(a, epsilon=1e-6, b=5, seed=1)
    assert f.row_indices == f2.row_indices and f.col_indices == f2.col_indices and t.status == t2.status


# ------------------------- round-2 fixes: QRCP rows on a permutation, sparse_nnz, wide blocks ------
@pytest.mark.parametrize("n,b", [(4, 2), (12, 5), (40, 33)])
def test_qrcp_rows_on_identity_matches_oracle(engine, oracle, n, b):
    """QRCP rows come in residual-norm order, not pivot order: D_k = A(I_k, J_k) can carry an exact
    zero on its diagonal (identity input, column pivots in descending order). The reference's COD
    (pinv.cpp:54-58) handles any nonsingular block; the engine factors D_k with partial pivoting."""
    a = np.eye(n)
    for seed in range(4):
        kw = dict(epsilon=1e-12, b=b, seed=seed, row_method="qrcp")
        f, t = engine.iterative_cur(a, **kw)
        o = oracle.iterative_cur(a, **kw)
        assert t.status == o.status and f.row_indices == o.row_indices and f.col_indices == o.col_indices
        assert all(math.isfinite(x) for x in t.rhos), t.rhos
        err = engine.true_relative_error(a, f)
        assert abs(err - oracle.true_relative_error(a, o.row_indices, o.col_indices)) <= 1e-8
        core = f.core_matrix()
        X = a[np.ix_(f.row_indices, f.col_indices)]
        assert np.allclose(core @ X, np.eye(f.rank), atol=1e-12)


def test_qrcp_rows_on_permuted_low_rank(engine, oracle):
    """Rows of a low-rank matrix shuffled so QRCP's row order differs from LUPP's: the pivoted
    D_k LU keeps I, J and the error equal to the oracle's."""
    rng = np.random.default_rng(5)
    a = low_rank_plus_noise(oracle, 300, 220, 40, 1e-11, 77)[rng.permutation(300)]
    kw = dict(epsilon=1e-9, b=12, seed=2, row_method="qrcp")
    f, t = engine.iterative_cur(a, **kw)
    o = oracle.iterative_cur(a, **kw)
    v = compare_runs(o, f, t)
    assert v["status_equal"] and v["identical"], v
    err = engine.true_relative_error(a, f)
    assert abs(err - oracle.true_relative_error(a, o.row_indices, o.col_indices)) <= 1e-8


def test_sparse_nnz_validation(engine, oracle):
    a = low_rank_plus_noise(oracle, 200, 150, 10, 1e-9, 3)
    with pytest.raises(ValueError, match="sparse_nnz must be at least 1"):
        engine.iterative_cur(a, b=20, sketch="sparse_sign", sparse_nnz=0)
    with pytest.raises(ValueError, match="sparse_nnz must be at least 1"):
        oracle.iterative_cur(a, b=20, sketch="sparse_sign", sparse_nnz=0)
    with pytest.raises(ValueError, match="sparse_nnz above 16"):
        engine.iterative_cur(a, b=20, sketch="sparse_sign", sparse_nnz=17)
    # min(zeta, c) is what the kernels draw: zeta = 40 with b = 10 (c = 11) is 11 slots, accepted
    kw = dict(epsilon=1e-6, b=10, seed=1, sketch="sparse_sign", sparse_nnz=40)
    f, t = engine.iterative_cur(a, **kw)
    o = oracle.iterative_cur(a, **kw)
    assert f.col_indices == o.col_indices and f.row_indices == o.row_indices


@pytest.mark.parametrize("b,sketch", [(250, "gaussian"), (200, "sparse_sign")])
def test_block_above_180_matches_oracle(engine, oracle, b, sketch):
    """b > 180 (the paper's runs use b = 250; the reference accepts any b <= m,
    driver.cpp:54): wide-block LUPP, cross LU and row solves with the factors in global memory."""
    # sigma_i = 10^(-i/60): tol 1e-5 stops near rank 300, pivots far above the rounding floor (a
    # low-rank-plus-1e-12-noise input would pick its last pivots from cancellation noise, H7)
    rng = np.random.default_rng(b)
    u, _ = np.linalg.qr(rng.standard_normal((1400, 1100)))
    v, _ = np.linalg.qr(rng.standard_normal((1100, 1100)))
    a = (u * 10.0 ** (-np.arange(1100) / 60.0)) @ v.T
    kw = dict(epsilon=1e-5, b=b, seed=4, sketch=sketch)
    f, t = engine.iterative_cur(a, **kw)
    o = oracle.iterative_cur(a, **kw)
    v = compare_runs(o, f, t)
    assert v["status_equal"] and v["identical"], v
    err = engine.true_relative_error(a, f)
    err_o = oracle.true_relative_error(a, o.row_indices, o.col_indices)
    assert abs(err - err_o) <= 1e-8, (err, err_o)
    core = f.core_matrix()
    X = a[np.ix_(f.row_indices, f.col_indices)]
    assert np.linalg.norm(core @ X - np.eye(f.rank)) <= 1e-7 * np.linalg.cond(X)


@pytest.mark.parametrize("rank", [500, 1000])
def test_slupp_large_rank_matches_oracle(engine, oracle, rank):
    """s-LUPP at the paper's sweep ranks (500-4000) runs as one engine block with b = r."""
    a = low_rank_plus_noise(oracle, 2500, 1600, 1200, 1e-8, 93)
    f = engine.slupp_cur(a, rank, 3)
    I, J = oracle.slupp_cur(a, rank, 3)
    assert f.rank == len(J)
    n_same = next((q for q in range(len(J)) if f.col_indices[q] != J[q] or f.row_indices[q] != I[q]), len(J))
    # one LUPP over rank pivots on a 1.1r-row sketch: the prefix is pinned until the first near tie
    assert n_same >= min(len(J), 100), n_same
    err = engine.true_relative_error(a, f)
    err_o = oracle.true_relative_error(a, I, J)
    assert abs(err - err_o) <= 1e-8 + 1e-3 * err_o, (err, err_o)


@pytest.mark.parametrize("b,sketch", [(50, "sparse_sign"), (64, "gaussian"), (40, "gaussian")])
def test_fused_wide_ublock_matches_oracle(engine, oracle, monkeypatch, b, sketch):
    """The fused U block for blocks 33..64 wide (opt-in ITERCUR_UB_MAX_N=64: U_k, the solves against
    D_k's LU with runtime pivot loops, R~_k and the downdate in one kernel) against the oracle."""
    monkeypatch.setenv("ITERCUR_UB_MAX_N", "64")
    a = low_rank_plus_noise(oracle, 1500, 1100, 220, 1e-10, 41 + b)
    kw = dict(epsilon=1e-8, b=b, seed=2, sketch=sketch)
    f, t = engine.iterative_cur(a, **kw)
    monkeypatch.delenv("ITERCUR_UB_MAX_N")
    f2, t2 = engine.iterative_cur(a, **kw)  # the unfused path
    o = oracle.iterative_cur(a, **kw)
    v = compare_runs(o, f, t)
    assert v["status_equal"] and v["identical"], v
    if v["full_identical"]:
        assert f.col_indices == f2.col_indices and np.allclose(t.rhos, t2.rhos, rtol=1e-9, atol=1e-13)
    err = engine.true_relative_error(a, f)
    assert abs(err - oracle.true_relative_error(a, o.row_indices, o.col_indices)) <= 1e-8


def test_preload_loads_every_engine_kernel(engine):
    """itercur_preload loads the kernels of all engine modules up front (lazy module loading would
    load each on its first launch inside the first iterative_cur call); runs still match after it."""
    n = engine.preload()
    assert n >= 100, n
    assert engine.preload() == n  # idempotent
    a = np.random.default_rng(3).standard_normal((300, 40)) @ np.random.default_rng(4).standard_normal((40, 250))
    f, t = engine.iterative_cur(a, epsilon=1e-10, b=10, seed=1)
    assert t.status in ("Converged", "ResidualExhausted") and 40 <= f.rank <= 50, (t.status, f.rank)

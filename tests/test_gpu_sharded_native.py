"""The native column-sharded engine (csrc/engine.cu) on one B200.

* Emulated shards (itercur_iterative_cur_sharded_emulated): S column shards computed by one process
  — per-shard sketch, U blocks, downdates and R~ columns, the selected block assembled from its
  owners, the replicated column/row selections — against the unsharded engine and the oracle.
* NCCL with one rank (itercur_iterative_cur_sharded_device over a communicator of size 1): every
  collective of the multi-rank path is issued (and captured in the iteration graphs).
Multi-rank NCCL needs several GPUs; the exchange protocol itself is covered on CPU with gloo
(tests/test_sharded_cpu.py)."""
import numpy as np
import pytest
import torch

from parity_util import compare_runs

pytestmark = pytest.mark.gpu


def lrn(oracle, m, n, r, rel, seed):
    a = oracle.random_gaussian(m, r, seed) @ oracle.random_gaussian(n, r, seed + 1).T
    g = oracle.random_gaussian(m, n, seed + 2)
    return a + (rel * np.linalg.norm(a) / np.linalg.norm(g)) * g


def decay(m, n, ratio, seed):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (u * ratio ** np.arange(n)) @ v.T


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda().t()


CASES = {
    "gauss_b10": (lambda o: lrn(o, 700, 530, 60, 1e-9, 3), dict(epsilon=1e-7, b=10, seed=1)),
    "sparse_b20": (lambda o: decay(900, 600, 0.97, 4), dict(epsilon=1e-4, b=20, seed=2, sketch="sparse_sign")),
    "gauss_b50_unfused": (lambda o: lrn(o, 1200, 900, 160, 1e-10, 5), dict(epsilon=1e-8, b=50, seed=3)),
    "sparse_b64": (lambda o: decay(1000, 800, 0.95, 6), dict(epsilon=1e-6, b=64, seed=4, sketch="sparse_sign")),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_emulated_shards_match_engine_and_oracle(engine, oracle, case, shards):
    from paper_2509_21963_b200.sharded import iterative_cur_emulated_shards

    make, kw = CASES[case]
    a = make(oracle)
    t = dev(a)
    f, tr = iterative_cur_emulated_shards(t, shards, **kw)
    f1, tr1 = engine.iterative_cur(engine.MatrixHandle.device(t), **kw)
    o = oracle.iterative_cur(a, **kw)
    v = compare_runs(o, f, tr)
    assert v["status_equal"] and v["identical"], (v, tr.status, o.status)
    assert tr.status == tr1.status
    if v["full_identical"]:
        assert f.col_indices == f1.col_indices and f.row_indices == f1.row_indices
        assert np.allclose(tr.rhos, tr1.rhos, rtol=1e-9, atol=1e-13)
    err = engine.true_relative_error(engine.MatrixHandle.device(t), f)
    err_o = oracle.true_relative_error(a, o.row_indices, o.col_indices)
    assert abs(err - err_o) <= 1e-8
    # every shard is local: the exports of the sharded run are the whole factors
    assert np.array_equal(f.c_matrix(), a[:, f.col_indices])
    core = f.core_matrix()
    X = a[np.ix_(f.row_indices, f.col_indices)]
    assert np.linalg.norm(core @ X - np.eye(f.rank)) <= 1e-10 * np.linalg.cond(X)


def test_emulated_shards_deterministic(engine, oracle):
    from paper_2509_21963_b200.sharded import iterative_cur_emulated_shards

    a = lrn(oracle, 800, 640, 70, 1e-9, 9)
    t = dev(a)
    runs = [iterative_cur_emulated_shards(t, 4, epsilon=1e-7, b=16, seed=5) for _ in range(3)]
    for f, tr in runs[1:]:
        assert f.col_indices == runs[0][0].col_indices and tr.rhos == runs[0][1].rhos


@pytest.mark.parametrize("kw", [dict(epsilon=1e-7, b=10, seed=1), dict(epsilon=1e-6, b=50, seed=2),
                                dict(epsilon=1e-4, b=20, seed=3, sketch="sparse_sign")])
def test_nccl_one_rank_matches_engine(engine, oracle, kw):
    from paper_2509_21963_b200.sharded import iterative_cur_sharded, shard_range, true_relative_error_sharded

    a = lrn(oracle, 900, 700, 120, 1e-10, 11)
    t = dev(a)
    assert shard_range(700, 1, 0) == (0, 700)
    res = iterative_cur_sharded(t, 0, 700, **kw)  # no process group: a communicator of one rank
    f1, tr1 = engine.iterative_cur(engine.MatrixHandle.device(t), **kw)
    assert res.status == tr1.status
    assert res.col_indices == f1.col_indices and res.row_indices == f1.row_indices
    assert np.allclose(res.rhos, tr1.rhos, rtol=1e-10, atol=1e-14)
    err = true_relative_error_sharded(t, 0, res)
    assert abs(err - engine.true_relative_error(engine.MatrixHandle.device(t), f1)) <= 1e-12
    with pytest.raises(RuntimeError, match="holds only its shard"):
        res.native.core_matrix()


def test_sharded_validation(engine, oracle):
    from paper_2509_21963_b200.sharded import iterative_cur_emulated_shards, shard_range

    a = lrn(oracle, 200, 160, 10, 1e-9, 13)
    t = dev(a)
    with pytest.raises(ValueError, match="LUPP selection only"):
        engine_sharded = iterative_cur_emulated_shards  # noqa: F841
        from paper_2509_21963_b200 import _capi, _config

        cfg = _config(1e-6, 8, 0.0, 0.05, False, 0, 0, "qrcp", "lupp", 1e-13, 0, "gaussian", 8, False)
        import ctypes as C

        out = C.c_void_p()
        _capi.check(_capi.lib().itercur_iterative_cur_sharded_emulated(C.c_void_p(t.data_ptr()), 200, 160, 200, 2,
                                                                       C.byref(cfg), None, C.byref(out)))
    with pytest.raises(ValueError, match="fewer than 2 columns"):
        iterative_cur_emulated_shards(t, 100, epsilon=1e-6, b=8)
    assert shard_range(101, 4, 3) == (78, 23) and shard_range(101, 4, 0) == (0, 26)

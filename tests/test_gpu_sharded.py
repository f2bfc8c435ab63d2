"""The column-sharded driver's per-rank stages on the B200 (sharded.DeviceBackend through the
C-ABI) against the test-only CPU backend and the oracle. Multi-rank exchanges are covered on
CPU with gloo (tests/test_sharded_cpu.py); one GPU here runs world_size 1."""
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sharded_cpu_backend import CpuBackend  # noqa: E402

pytestmark = pytest.mark.gpu


def _dev():
    from paper_2509_21963_b200.sharded import DeviceBackend
    return DeviceBackend("cuda:0")


def test_dist_lupp_steps_bit_exact_vs_cpu():
    from paper_2509_21963_b200.sharded import to_colmajor
    rng = np.random.default_rng(4)
    rows, steps = 3000, 12
    w0 = torch.from_numpy(rng.standard_normal((rows, steps)))
    live0 = torch.ones(rows, dtype=torch.uint8)
    live0[::7] = 0
    dev, cpu = _dev(), CpuBackend()
    Wd, Wc = to_colmajor(w0.cuda()), to_colmajor(w0.clone())
    ld, lc = live0.cuda(), live0.clone()
    cd = torch.zeros(4 + steps, dtype=torch.float64, device="cuda")
    cc = torch.zeros(4 + steps, dtype=torch.float64)
    P = None
    piv = -1
    for s in range(steps):
        dev.lupp_step(Wd, ld, steps, s, P.cuda() if P is not None else None, piv, 100, cd)
        cpu.lupp_step(Wc, lc, steps, s, P, piv, 100, cc)
        torch.cuda.synchronize()
        assert torch.equal(cd.cpu(), cc), (s, cd.cpu(), cc)
        P = cc[4:].clone()
        piv = int(cc[2]) - 100
    assert torch.equal(Wd.cpu(), Wc)


def test_gemm_block_lu_and_solves():
    from paper_2509_21963_b200.sharded import to_colmajor
    rng = np.random.default_rng(5)
    dev, cpu = _dev(), CpuBackend()
    A = torch.from_numpy(rng.standard_normal((1000, 77)))
    B = torch.from_numpy(rng.standard_normal((77, 19)))
    base = torch.from_numpy(rng.standard_normal((1000, 19)))
    out = to_colmajor(torch.empty(1000, 19, dtype=torch.float64, device="cuda"))
    dev.gemm(to_colmajor(A.cuda()), to_colmajor(B.cuda()), to_colmajor(base.cuda()), -1.0, out)
    ref = base - A @ B
    assert torch.allclose(out.cpu(), ref, rtol=0, atol=1e-12 * float(ref.abs().max()))
    D0 = torch.from_numpy(rng.standard_normal((13, 13)) + 13 * np.eye(13))
    Dd = to_colmajor(D0.cuda())
    dev.block_lu(Dd)
    Dc = cpu.block_lu(to_colmajor(D0.clone()))
    assert torch.equal(Dd.cpu(), Dc)  # same operations, same order
    X = torch.from_numpy(rng.standard_normal((500, 13)))
    od = to_colmajor(torch.empty(500, 13, dtype=torch.float64, device="cuda"))
    dev.rows_solve(to_colmajor(X.cuda()), Dd, od)
    x_ref = torch.linalg.solve(D0, X.T).T
    assert torch.allclose(od.cpu(), x_ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kw", [dict(epsilon=1e-8, b=5, seed=2), dict(epsilon=1e-6, b=8, seed=1, sketch="sparse_sign"),
                                dict(epsilon=0.0, b=4, seed=3, max_rank=10)])
@pytest.mark.parametrize("exchange", ["sketch", "candidates"])
def test_world_one_on_the_gpu_matches_oracle(oracle, kw, exchange):
    from paper_2509_21963_b200.sharded import iterative_cur_sharded, true_relative_error_sharded
    a = oracle.random_gaussian(300, 20, 5) @ oracle.random_gaussian(240, 20, 6).T
    a = a + 1e-9 * np.linalg.norm(a) / 300.0 * oracle.random_gaussian(300, 240, 7)
    o = oracle.iterative_cur(a, **kw)
    t = torch.from_numpy(np.asfortranarray(a)).cuda()
    t = t.t().contiguous().t()
    res = iterative_cur_sharded(t, 0, a.shape[1], column_exchange=exchange, **kw)
    assert res.status == o.status
    assert res.row_indices == list(o.row_indices) and res.col_indices == list(o.col_indices)
    err = true_relative_error_sharded(t, 0, res)
    err_o = oracle.true_relative_error(a, o.row_indices, o.col_indices)
    assert abs(err - err_o) <= 1e-8

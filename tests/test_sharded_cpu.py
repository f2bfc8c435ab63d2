"""The column-sharded driver (paper_2509_21963_b200/sharded.py) on CPU:
world_size 2 over gloo with the test-only torch/oracle backend, against the single-process
oracle (proj/src/driver.cpp:48-167 restated). The product path runs the same driver with the
B200 kernels (tests/test_gpu_sharded.py)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sharded_cpu_backend import CpuBackend  # noqa: E402

from paper_2509_21963_b200.sharded import iterative_cur_sharded, true_relative_error_sharded  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cases(oracle):
    rng = np.random.default_rng(3)
    # low rank + noise, odd column split
    a1 = oracle.random_gaussian(120, 12, 5) @ oracle.random_gaussian(90, 12, 6).T
    a1 = a1 + 1e-9 * np.linalg.norm(a1) / 100.0 * oracle.random_gaussian(120, 90, 7)
    # exponential decay spectrum
    n = 80
    q1, _ = np.linalg.qr(rng.standard_normal((100, n)))
    q2, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a2 = (q1 * 0.8 ** np.arange(n)) @ q2.T
    return {
        "lowrank_noise": (a1, dict(epsilon=1e-8, b=5, seed=2)),
        "expdecay_sparse_sign": (a2, dict(epsilon=1e-5, b=6, seed=1, sketch="sparse_sign")),
        "fixed_rank": (a1, dict(epsilon=0.0, b=4, seed=3, max_rank=10)),
    }


def _worker(rank, world, port, case, out_q, exchange="sketch"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        a, kw = _cases(oracle)[case]
        n = a.shape[1]
        bounds = [round(q * n / world) for q in range(world + 1)]
        lo, hi = bounds[rank], bounds[rank + 1]
        shard = torch.from_numpy(np.asfortranarray(a[:, lo:hi]))
        res = iterative_cur_sharded(shard, lo, n, backend=CpuBackend(), column_exchange=exchange, **kw)
        err = true_relative_error_sharded(shard, lo, res)
        out_q.put((rank, res.row_indices, res.col_indices, res.status, res.final_rho, err, res.exchanges))
    finally:
        dist.destroy_process_group()


def _run(case, world, exchange="sketch"):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, exchange)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    outs = sorted(q.get() for _ in range(world))
    return outs


@pytest.mark.parametrize("exchange", ["sketch", "candidates"])
@pytest.mark.parametrize("case", ["lowrank_noise", "expdecay_sparse_sign", "fixed_rank"])
def test_two_ranks_match_single_process_oracle(oracle, case, exchange):
    a, kw = _cases(oracle)[case]
    o = oracle.iterative_cur(a, **kw)
    outs = _run(case, 2, exchange)
    # every rank returns the same selection
    assert outs[0][1:5] == outs[1][1:5]
    _, I, J, status, rho, err, exchanges = outs[0]
    assert status == o.status
    assert I == list(o.row_indices) and J == list(o.col_indices)
    assert abs(rho - o.final_rho) <= 1e-9 + 1e-6 * o.final_rho
    err_o = oracle.true_relative_error(a, o.row_indices, o.col_indices)
    assert abs(err - err_o) <= 1e-8
    assert exchanges > 0


def test_single_process_without_distributed(oracle):
    a, kw = _cases(oracle)["lowrank_noise"]
    o = oracle.iterative_cur(a, **kw)
    res = iterative_cur_sharded(torch.from_numpy(np.asfortranarray(a)), 0, a.shape[1], backend=CpuBackend(), **kw)
    assert res.row_indices == list(o.row_indices) and res.col_indices == list(o.col_indices)
    assert res.status == o.status and res.exchanges == 0


def test_validation_messages(oracle):
    a = oracle.random_dense(4, 6, 1)
    t = torch.from_numpy(np.asfortranarray(a))
    with pytest.raises(ValueError, match="block exceeds row count"):
        iterative_cur_sharded(t, 0, 6, b=5, backend=CpuBackend())
    with pytest.raises(ValueError, match="nonzero"):
        iterative_cur_sharded(torch.zeros(4, 6, dtype=torch.float64), 0, 6, b=2, backend=CpuBackend())
    with pytest.raises(ValueError, match="contiguous column ranges"):
        iterative_cur_sharded(t, 1, 6, b=2, backend=CpuBackend())

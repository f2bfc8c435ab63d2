"""The reference's own Python smoke tests (proj/tests/python/test_smoke.py:36-52,78-84) restated under
INTEGRATION.md §2's import switch: `iterative_cur` / `true_relative_error` come from the B200 engine
while the matrices stay the reference's `MatrixHandle` objects (`itercur.low_rank(...)`,
`MatrixHandle.dense(...)`).

The reference's compiled `_itercur` module cannot be built here (no Eigen), so
`RefHandle` stands in for its pybind11 MatrixHandle with exactly the surface module.cpp:36-57
exposes (rows / cols / is_sparse / nnz / to_numpy / fro_norm) — the engine sees nothing else."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class RefHandle:
    """The reference binding's MatrixHandle surface (module.cpp:36-57); not a numpy array."""

    def __init__(self, array):
        self._a = np.array(array, dtype=np.float64)

    @staticmethod
    def dense(array):
        return RefHandle(array)

    rows = property(lambda self: self._a.shape[0])
    cols = property(lambda self: self._a.shape[1])
    is_sparse = property(lambda self: False)
    nnz = property(lambda self: self._a.size)

    def to_numpy(self):
        return self._a.copy()

    def fro_norm(self):
        return float(np.linalg.norm(self._a))


def low_rank(oracle, m, n, r, seed=0):
    """itercur.low_rank (GeneratorSpec::low_rank, testmat.cpp:19-49): a rank-r product, as a handle."""
    return RefHandle(oracle.random_gaussian(m, r, seed) @ oracle.random_gaussian(n, r, seed + 1).T)


class itercur:  # noqa: N801  (the switched namespace of INTEGRATION.md §2)
    from paper_2509_21963_b200 import iterative_cur, true_relative_error  # noqa: F401

    MatrixHandle = RefHandle


def test_iterative_cur_recovers_exact_rank(oracle):  # test_smoke.py:36-43
    a = low_rank(oracle, 120, 100, 8, seed=3)
    factors, trace = itercur.iterative_cur(a, epsilon=1e-8, b=4, seed=7)
    assert trace.status == "Converged"
    assert factors.rank == 8
    assert len(factors.row_indices) == len(factors.col_indices) == 8
    assert itercur.true_relative_error(a, factors) <= 1e-10
    assert trace.rhos[-1] == pytest.approx(trace.final_rho)


def test_factors_reconstruct_the_matrix(oracle):  # test_smoke.py:46-52
    a = low_rank(oracle, 40, 30, 5, seed=1)
    factors, _ = itercur.iterative_cur(a, epsilon=1e-8, b=5, seed=2)
    dense = a.to_numpy()
    approx = factors.c_matrix() @ factors.core_matrix() @ factors.r_matrix()
    rel = np.linalg.norm(dense - approx) / np.linalg.norm(dense)
    assert rel <= 1e-9


def test_zero_matrix_is_rejected():  # test_smoke.py:78-84
    zero = itercur.MatrixHandle.dense(np.zeros((4, 4)))
    with pytest.raises(ValueError):
        itercur.iterative_cur(zero, epsilon=1e-3, b=2)


def test_true_relative_error_uses_the_given_matrix(engine, oracle):
    """true_relative_error(A, factors) evaluates the matrix it is given (driver.cpp:169-190),
    host or device, against the run's factors — also after the host entry freed its copy of A."""
    import torch

    a = oracle.random_gaussian(300, 20, 7) @ oracle.random_gaussian(250, 20, 8).T
    f, t = engine.iterative_cur(a, epsilon=1e-9, b=10, seed=1)
    err = engine.true_relative_error(a, f)
    assert err <= 1e-10
    b = a.copy()
    b[:, 3] += 1.0
    err_b = engine.true_relative_error(b, f)
    x = a[np.ix_(f.row_indices, f.col_indices)]
    direct = np.linalg.norm(b - a[:, f.col_indices] @ np.linalg.solve(x, a[f.row_indices, :])) / np.linalg.norm(b)
    assert err_b == pytest.approx(direct, rel=1e-9) and err_b > 1e-3
    t_b = torch.from_numpy(np.ascontiguousarray(b.T)).cuda().t()
    assert engine.true_relative_error(engine.MatrixHandle.device(t_b), f) == pytest.approx(err_b, rel=1e-12)
    with pytest.raises(ValueError, match="factors are for"):
        engine.true_relative_error(np.ones((5, 5)), f)


def test_observer_sees_every_iteration(engine, oracle):
    a = oracle.random_gaussian(200, 30, 3) @ oracle.random_gaussian(160, 30, 4).T
    seen = []

    def obs(f, rec):
        c = f.c_matrix()
        assert np.array_equal(c, a[:, f.col_indices])
        core = f.core_matrix()
        x = a[np.ix_(f.row_indices, f.col_indices)]
        assert np.allclose(core @ x, np.eye(f.rank), atol=1e-8)
        seen.append((rec.k, f.rank, rec.rho))

    f, t = engine.iterative_cur(a, epsilon=1e-10, b=6, seed=2, observer=obs)
    assert [s[0] for s in seen] == list(range(len(t.iterations)))
    assert seen[-1][1] == f.rank and [s[2] for s in seen] == t.rhos
    f2, t2 = engine.iterative_cur(a, epsilon=1e-10, b=6, seed=2)  # same run without the observer
    assert f2.col_indices == f.col_indices and t2.rhos == t.rhos

    def boom(f, rec):
        raise KeyError("stop here")

    with pytest.raises(KeyError, match="stop here"):
        engine.iterative_cur(a, epsilon=1e-10, b=6, seed=2, observer=boom)


def test_row_pivot_floor_is_per_method(engine, oracle):
    a = oracle.random_gaussian(200, 40, 3) @ oracle.random_gaussian(160, 40, 4).T
    f, t = engine.iterative_cur(a, epsilon=1e-10, b=8, seed=2, row_pivot_floor=0.99)
    # the row floor truncates the first row block; the column block (default floor) is full
    assert t.iterations[0].row_truncated and not t.iterations[0].col_truncated
    with pytest.raises(ValueError, match="pivot_floor"):
        engine.iterative_cur(a, b=8, row_pivot_floor=2.0)


def test_host_entry_releases_the_device_copy(engine, oracle):
    import torch

    a = oracle.random_gaussian(3000, 40, 3) @ oracle.random_gaussian(2000, 40, 4).T
    torch.cuda.synchronize()
    f, t = engine.iterative_cur(a, epsilon=1e-10, b=20, seed=2)
    L = engine._lib()
    assert L.itercur_run_holds_matrix(f._run.ptr) == 0
    assert np.array_equal(f.c_matrix(), a[:, f.col_indices])
    assert np.array_equal(f.r_matrix(), a[f.row_indices, :])
    assert engine.sketched_relative_error(a, f, 20, 2) == pytest.approx(t.final_rho, abs=1e-12)

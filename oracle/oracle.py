"""ctypes wrapper over oracle/liboracle.so — the CPU ORACLE (test infrastructure).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) import this module, and only as the checker / timed CPU
baseline. The product (``paper_2509_21963_b200``) never imports it.

The library restates /root/reference/proj/src/{rng,sketch,select,pinv,matrix,driver}.cpp;
see oracle/itercur_oracle.h for the pinning status of each piece.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, E_INVALID, E_RANGE, E_DOMAIN, E_RUNTIME, E_LOGIC = range(6)
STATUS_NAMES = {0: "Converged", 1: "MaxRank", 2: "ResidualExhausted"}
SKETCH_KINDS = {"gaussian": 0, "sparse_sign": 1}
METHODS = {"lupp": 0, "qrcp": 1, "osinsky": 2}
STREAM_SKETCH = 1
STREAM_SPARSE_SIGN = 7


class _Config(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double), ("b", C.c_int64), ("delta", C.c_double), ("alpha", C.c_double),
        ("risk_adjust", C.c_int32), ("max_rank", C.c_int64), ("max_iters", C.c_int64),
        ("col_method", C.c_int32), ("row_method", C.c_int32), ("pivot_floor", C.c_double),
        ("seed", C.c_uint64), ("sketch_kind", C.c_int32), ("sparse_nnz", C.c_int32),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("cap_rank", C.c_int64), ("row_indices", C.POINTER(C.c_int64)), ("col_indices", C.POINTER(C.c_int64)),
        ("cap_iters", C.c_int64), ("rhos", C.POINTER(C.c_double)), ("widths", C.POINTER(C.c_int64)),
        ("iter_seconds", C.POINTER(C.c_double)),
        ("cap_steps", C.c_int64), ("step_kind", C.POINTER(C.c_int32)), ("step_iter", C.POINTER(C.c_int64)),
        ("step_index", C.POINTER(C.c_int64)), ("step_best", C.POINTER(C.c_double)),
        ("step_second", C.POINTER(C.c_double)),
        ("rank", C.c_int64), ("n_iters", C.c_int64), ("n_steps", C.c_int64), ("status", C.c_int32),
        ("final_rho", C.c_double), ("threshold", C.c_double), ("sketch_s", C.c_double), ("total_s", C.c_double),
        ("ga_norm", C.c_double), ("c", C.c_int64), ("note", C.c_char * 128),
        ("cod_rank", C.POINTER(C.c_int64)),
    ]


def build(quiet: bool = True) -> None:
    """Compile the oracle with its Makefile (and oracle/_ref when /root/reference exists)."""
    targets = ["all"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-C", _HERE, *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        dp, i64p = C.POINTER(C.c_double), C.POINTER(C.c_int64)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_normal_at.restype = C.c_double
        L.oracle_normal_at.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64]
        L.oracle_uniform_at.restype = C.c_double
        L.oracle_uniform_at.argtypes = [C.c_uint64, C.c_uint32, C.c_int64, C.c_int64]
        L.oracle_gaussian_matrix.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_uint32, dp]
        L.oracle_set_threads.argtypes = [C.c_int]
        L.oracle_set_threads.restype = C.c_int
        L.oracle_gaussian_fill.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_uint32, C.c_double, dp]
        L.oracle_philox4x32.argtypes = [C.POINTER(C.c_uint32)] * 3
        L.oracle_sparse_sign_pattern.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int32,
                                                 C.POINTER(C.c_int32), C.POINTER(C.c_int8)]
        L.oracle_sketch_rows_for_block.restype = C.c_int64
        L.oracle_sketch_rows_for_block.argtypes = [C.c_int64]
        L.oracle_sketch.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int32,
                                    C.c_int32, dp, dp, dp]
        L.oracle_select.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                    C.c_double, i64p, C.c_int64, i64p, i64p, C.POINTER(C.c_int32), dp, dp, dp]
        L.oracle_adjusted_threshold.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64, dp]
        L.oracle_gratton_tail.argtypes = [C.c_int64, C.c_double, dp]
        L.oracle_iterative_cur.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, C.POINTER(_Config),
                                           C.POINTER(_Result)]
        L.oracle_true_relative_error.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, i64p, i64p, C.c_int64, dp]
        L.oracle_core_matrix.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, i64p, i64p, C.c_int64, dp]
        L.oracle_core_solve.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, i64p, i64p, C.c_int64, dp, C.c_int64,
                                        C.c_int64, dp]
        L.oracle_slupp_cur.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, i64p, i64p,
                                       C.POINTER(C.c_int64)]
        L.oracle_fixture_random_dense.argtypes = [C.c_int64, C.c_int64, C.c_uint32, C.c_double, C.c_double, dp]
        L.oracle_fixture_random_gaussian.argtypes = [C.c_int64, C.c_int64, C.c_uint32, dp]
        _lib = L
    return _lib


class OracleError(Exception):
    pass


_EXC = {E_INVALID: ValueError, E_RANGE: IndexError, E_DOMAIN: ValueError, E_RUNTIME: RuntimeError,
        E_LOGIC: RuntimeError}


def _check(rc: int) -> None:
    if rc != OK:
        msg = lib().oracle_last_error().decode()
        raise _EXC.get(rc, OracleError)(msg)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _colmajor(a: np.ndarray) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ----------------------------------------------------------------------- fixtures
def random_dense(rows, cols, seed, lo=-1.0, hi=1.0) -> np.ndarray:
    """proj/tests/oracles.hpp:20-28 (mt19937_64 + uniform_real_distribution, column order)."""
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    lib().oracle_fixture_random_dense(rows, cols, seed, lo, hi, _dp(out))
    return out


def random_gaussian(rows, cols, seed) -> np.ndarray:
    """proj/tests/oracles.hpp:30-37 (mt19937_64 + normal_distribution, column order)."""
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    lib().oracle_fixture_random_gaussian(rows, cols, seed, _dp(out))
    return out


# ---------------------------------------------------------------------------- rng
def philox4x32(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    out = (C.c_uint32 * 4)()
    lib().oracle_philox4x32(c, k, out)
    return list(out)


def normal_at(seed, stream, i, j) -> float:
    return lib().oracle_normal_at(seed, stream, i, j)


def uniform_at(seed, stream, i, j) -> float:
    return lib().oracle_uniform_at(seed, stream, i, j)


def gaussian_matrix(rows, cols, seed, stream=STREAM_SKETCH) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    lib().oracle_gaussian_matrix(rows, cols, seed, stream, _dp(out))
    return out


def set_threads(n: int) -> int:
    """Threads for the oracle's column-parallel loops (0 = all); returns the count in use."""
    return int(lib().oracle_set_threads(int(n)))


def gaussian_fill(out: np.ndarray, seed, stream, scale=1.0) -> None:
    """out(i, j) = scale * normal_at(seed, stream, i, j) in place (Fortran-ordered float64; threaded)."""
    assert out.dtype == np.float64 and out.flags.f_contiguous and out.ndim == 2
    rows, cols = out.shape
    lib().oracle_gaussian_fill(rows, cols, max(rows, 1), seed, stream, scale, _dp(out))


def sparse_sign_pattern(c, m, seed, zeta=8):
    ze = min(zeta, c)
    rows = np.empty((m, ze), dtype=np.int32)
    signs = np.empty((m, ze), dtype=np.int8)
    _check(lib().oracle_sparse_sign_pattern(c, m, seed, zeta, rows.ctypes.data_as(C.POINTER(C.c_int32)),
                                            signs.ctypes.data_as(C.POINTER(C.c_int8))))
    return rows, signs


def sketch_rows_for_block(b: int) -> int:
    return lib().oracle_sketch_rows_for_block(b)


def sketch(a, b, seed, kind="gaussian", zeta=8):
    """(Y = S*A (c x n), ||Y||_F, ||A||_F) — proj/src/sketch.cpp:10-24."""
    a = _colmajor(a)
    m, n = a.shape
    c = sketch_rows_for_block(b)
    y = np.zeros((max(c, 0), n), dtype=np.float64, order="F")
    ga, an = C.c_double(), C.c_double()
    _check(lib().oracle_sketch(_dp(a), m, n, max(m, 1), b, seed, SKETCH_KINDS[kind], zeta, _dp(y),
                               C.byref(ga), C.byref(an)))
    return y, ga.value, an.value


# ---------------------------------------------------------------------- selection
@dataclass
class Selection:
    indices: list
    truncated: bool
    last_pivot_magnitude: float
    best: list = field(default_factory=list)
    second: list = field(default_factory=list)


def _select(m, b, is_columns, method, pivot_floor, exclude):
    m = _colmajor(m)
    rows, cols = m.shape
    ex = np.asarray(list(exclude), dtype=np.int64)
    cap = max(b, 1) + 1
    idx = np.zeros(cap, dtype=np.int64)
    best = np.zeros(cap)
    second = np.zeros(cap)
    nidx = C.c_int64()
    trunc = C.c_int32()
    last = C.c_double()
    _check(lib().oracle_select(_dp(m), rows, cols, max(rows, 1), b, 1 if is_columns else 0, METHODS[method],
                               pivot_floor, _i64p(ex), len(ex), _i64p(idx), C.byref(nidx), C.byref(trunc),
                               C.byref(last), _dp(best), _dp(second)))
    k = nidx.value
    return Selection([int(v) for v in idx[:k]], bool(trunc.value), last.value, list(best[:k]), list(second[:k]))


def select_columns(m, b, method="lupp", pivot_floor=1e-13, exclude=()):
    return _select(m, b, True, method, pivot_floor, exclude)


def select_rows(m, b, method="lupp", pivot_floor=1e-13, exclude=()):
    return _select(m, b, False, method, pivot_floor, exclude)


# ------------------------------------------------------------------------- driver
def adjusted_threshold(epsilon, delta, alpha, c) -> float:
    out = C.c_double()
    _check(lib().oracle_adjusted_threshold(epsilon, delta, alpha, c, C.byref(out)))
    return out.value


def gratton_tail(c, tau) -> float:
    out = C.c_double()
    _check(lib().oracle_gratton_tail(c, tau, C.byref(out)))
    return out.value


@dataclass
class OracleRun:
    row_indices: list
    col_indices: list
    status: str
    final_rho: float
    threshold: float
    rhos: list
    widths: list
    note: str
    sketch_s: float
    total_s: float
    ga_norm: float
    c: int
    steps: list  # (kind, iteration, index, best, second)
    iter_seconds: list = field(default_factory=list)
    cod_ranks: list = field(default_factory=list)  # per iteration: numerical rank of the core's COD

    @property
    def rank(self) -> int:
        return len(self.col_indices)


def iterative_cur(a, epsilon=1e-6, b=50, delta=0.0, alpha=0.05, risk_adjust=False, max_rank=0, max_iters=0,
                  col_method="lupp", row_method="lupp", pivot_floor=1e-13, seed=0, sketch="gaussian",
                  sparse_nnz=8, log_steps=True) -> OracleRun:
    """proj/src/driver.cpp:48-167 restated; returns indices, trace and per-pivot margins."""
    a = _colmajor(a)
    m, n = a.shape
    cfg = _Config(epsilon, b, delta, alpha, 1 if risk_adjust else 0, max_rank, max_iters, METHODS[col_method],
                  METHODS[row_method], pivot_floor, seed, SKETCH_KINDS[sketch], sparse_nnz)
    cap_rank = max(min(m, n), 1)
    cap_iters = (min(m, n) + max(b, 1) - 1) // max(b, 1) + 2 if max_iters <= 0 else max_iters + 1
    cap_steps = 2 * cap_rank + 2 * b + 8 if log_steps else 0
    I = np.zeros(cap_rank, dtype=np.int64)
    J = np.zeros(cap_rank, dtype=np.int64)
    rhos = np.zeros(cap_iters)
    widths = np.zeros(cap_iters, dtype=np.int64)
    iter_s = np.zeros(cap_iters)
    sk = np.zeros(max(cap_steps, 1), dtype=np.int32)
    si = np.zeros(max(cap_steps, 1), dtype=np.int64)
    sx = np.zeros(max(cap_steps, 1), dtype=np.int64)
    sb = np.zeros(max(cap_steps, 1))
    ss = np.zeros(max(cap_steps, 1))
    res = _Result()
    res.cap_rank, res.row_indices, res.col_indices = cap_rank, _i64p(I), _i64p(J)
    res.cap_iters, res.rhos, res.widths = cap_iters, _dp(rhos), _i64p(widths)
    res.iter_seconds = _dp(iter_s)
    cod = np.zeros(cap_iters, dtype=np.int64)
    res.cod_rank = _i64p(cod)
    res.cap_steps = cap_steps
    res.step_kind = sk.ctypes.data_as(C.POINTER(C.c_int32))
    res.step_iter, res.step_index, res.step_best, res.step_second = _i64p(si), _i64p(sx), _dp(sb), _dp(ss)
    _check(lib().oracle_iterative_cur(_dp(a), m, n, max(m, 1), C.byref(cfg), C.byref(res)))
    r, k = res.rank, res.n_iters
    nst = min(res.n_steps, cap_steps)
    steps = [(int(sk[q]), int(si[q]), int(sx[q]), float(sb[q]), float(ss[q])) for q in range(nst)]
    return OracleRun([int(v) for v in I[:r]], [int(v) for v in J[:r]], STATUS_NAMES[res.status], res.final_rho,
                     res.threshold, list(rhos[:k]), [int(v) for v in widths[:k]], res.note.decode(),
                     res.sketch_s, res.total_s, res.ga_norm, res.c, steps, list(iter_s[:k]),
                     [int(v) for v in cod[:k]])


def slupp_cur(a, rank, seed=0):
    """One-shot s-LUPP CUR baseline (proj/src/baselines.cpp:39-62): (row_indices, col_indices)."""
    a = _colmajor(a)
    m, n = a.shape
    cap = max(int(rank), 1)
    I = np.zeros(cap, dtype=np.int64)
    J = np.zeros(cap, dtype=np.int64)
    k = C.c_int64()
    _check(lib().oracle_slupp_cur(_dp(a), m, n, max(m, 1), int(rank), int(seed), _i64p(I), _i64p(J), C.byref(k)))
    return [int(v) for v in I[:k.value]], [int(v) for v in J[:k.value]]


def true_relative_error(a, row_indices, col_indices) -> float:
    a = _colmajor(a)
    m, n = a.shape
    I = np.asarray(row_indices, dtype=np.int64)
    J = np.asarray(col_indices, dtype=np.int64)
    out = C.c_double()
    _check(lib().oracle_true_relative_error(_dp(a), m, n, max(m, 1), _i64p(I), _i64p(J), len(I), C.byref(out)))
    return out.value


def core_matrix(a, row_indices, col_indices) -> np.ndarray:
    a = _colmajor(a)
    m, n = a.shape
    I = np.asarray(row_indices, dtype=np.int64)
    J = np.asarray(col_indices, dtype=np.int64)
    r = len(I)
    out = np.zeros((r, r), dtype=np.float64, order="F")
    _check(lib().oracle_core_matrix(_dp(a), m, n, max(m, 1), _i64p(I), _i64p(J), r, _dp(out)))
    return out


def core_solve(a, row_indices, col_indices, rhs) -> np.ndarray:
    """A(I,J)^+ @ rhs by the oracle's COD minimum-norm solve (proj/src/pinv.cpp:24-31)."""
    a = _colmajor(a)
    m, n = a.shape
    I = np.asarray(row_indices, dtype=np.int64)
    J = np.asarray(col_indices, dtype=np.int64)
    rhs = _colmajor(rhs)
    r, k = rhs.shape
    assert r == len(I) == len(J)
    out = np.zeros((r, k), dtype=np.float64, order="F")
    _check(lib().oracle_core_solve(_dp(a), m, n, max(m, 1), _i64p(I), _i64p(J), r, _dp(rhs), k, max(r, 1), _dp(out)))
    return out

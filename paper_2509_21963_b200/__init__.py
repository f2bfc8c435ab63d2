"""B200-native IterativeCUR — drop-in for the reference's ``itercur`` hot path.

Mirrors the Python surface of the reference binding (proj/bindings/python/module.cpp:34-163,
re-exported by proj/python/itercur/__init__.py:3-43) for the IterativeCUR path:

    factors, trace = iterative_cur(a, epsilon=1e-6, b=50, delta=0.0, alpha=0.05,
                                   risk_adjust=False, max_rank=0, max_iters=0,
                                   col_method="lupp", row_method="lupp",
                                   pivot_floor=1e-13, seed=0)

plus the new ``sketch="gaussian" | "sparse_sign"`` and ``sparse_nnz`` keywords. Everything
runs through the C-ABI in include/itercur_b200.h (libitercur_b200.so, hand-written
sm_100a kernels); there is no CPU fallback. Exceptions follow pybind11's mapping of the
reference's C++ exceptions (invalid_argument/domain_error -> ValueError,
out_of_range -> IndexError, runtime_error -> RuntimeError).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check as _check

__version__ = "0.1.0"

_METHODS = {"lupp": 0, "qrcp": 1, "osinsky": 2}
_SKETCHES = {"gaussian": 0, "sparse_sign": 1}
_STATUS = {0: "Converged", 1: "MaxRank", 2: "ResidualExhausted"}


def _lib():
    return _capi.lib()


# ------------------------------------------------------------------------- matrices
class MatrixHandle:
    """Dense column-major FP64 matrix (proj/include/itercur/matrix.hpp:27-59, dense path).

    ``MatrixHandle.dense(array)`` keeps a host copy (the reference copies numpy into Eigen,
    module.cpp:38-39) and rejects non-finite entries (matrix.cpp:73-77).
    ``MatrixHandle.device(tensor)`` wraps a CUDA tensor in place (no host round trip): a
    torch.float64 tensor of shape (m, n) with column-major strides (1, lda), e.g.
    ``torch.empty(n, m, device="cuda", dtype=torch.float64).t()``.
    """

    def __init__(self, host=None, tensor=None, csr=None, shape=None):
        self._host = host
        self._tensor = tensor
        self._csr = csr  # (row_ptr, col_idx, values) int64 / int64 / float64 numpy arrays
        if host is not None:
            self.rows, self.cols = host.shape
        elif tensor is not None:
            self.rows, self.cols = int(tensor.shape[0]), int(tensor.shape[1])
        else:
            self.rows, self.cols = shape

    @staticmethod
    def sparse_csr(rows, cols, indptr, indices, data) -> "MatrixHandle":
        """CSR matrix (binding module.cpp:40-48 -> matrix.cpp:79-104), validated as the
        reference validates it. The engine densifies it on the device before a run."""
        rows, cols = int(rows), int(cols)
        if rows < 0 or cols < 0:
            raise ValueError("negative matrix dimension")
        rp = np.asarray(indptr, dtype=np.int64)
        ci = np.asarray(indices, dtype=np.int64)
        v = np.asarray(data, dtype=np.float64)
        if rp.shape != (rows + 1,):
            raise ValueError("row_ptr must have rows+1 entries")
        if rp[0] != 0 or rp[-1] != v.size:
            raise ValueError("row_ptr must start at 0 and end at nnz")
        if ci.size != v.size:
            raise ValueError("col_idx and values must have equal length")
        if np.any(np.diff(rp) < 0):
            raise ValueError("row_ptr must be nondecreasing")
        bad = np.nonzero((ci < 0) | (ci >= cols))[0]
        if bad.size:
            raise IndexError(f"csr column index {int(ci[bad[0]])} out of range [0, {cols})")
        for i in range(rows):
            seg = ci[rp[i]:rp[i + 1]]
            if seg.size > 1 and np.any(np.diff(seg) <= 0):
                raise ValueError("csr column indices must be strictly increasing within each row")
        if not np.all(np.isfinite(v)):
            raise ValueError("matrix contains non-finite entries")
        return MatrixHandle(csr=(rp, ci, v), shape=(rows, cols))

    def _densified_on_device(self) -> "MatrixHandle":
        """The CSR matrix scattered into a dense column-major device buffer (B200 kernel)."""
        import torch

        rp, ci, v = (torch.from_numpy(x).cuda() for x in self._csr)
        out = torch.empty(max(self.cols, 1), max(self.rows, 1), dtype=torch.float64, device="cuda").t()
        out = out[:self.rows, :self.cols]
        stream = torch.cuda.current_stream().cuda_stream
        _check(_lib().itercur_csr_to_dense_device(self.rows, self.cols, C.c_void_p(rp.data_ptr()),
                                                  C.c_void_p(ci.data_ptr()), C.c_void_p(v.data_ptr()),
                                                  C.c_void_p(out.data_ptr()), max(self.rows, 1), C.c_void_p(stream)))
        return MatrixHandle(tensor=out)

    @staticmethod
    def dense(array) -> "MatrixHandle":
        a = np.asfortranarray(np.asarray(array, dtype=np.float64))
        if a.ndim != 2:
            raise ValueError("dense matrix must be two-dimensional")
        if not _all_finite(a):
            raise ValueError("matrix contains non-finite entries")
        return MatrixHandle(host=a)

    @staticmethod
    def device(tensor) -> "MatrixHandle":
        import torch  # device memory / streams are torch's; the engine only sees pointers

        if not isinstance(tensor, torch.Tensor) or not tensor.is_cuda or tensor.dtype != torch.float64:
            raise ValueError("MatrixHandle.device expects a float64 CUDA tensor")
        if tensor.dim() != 2:
            raise ValueError("device matrix must be two-dimensional")
        m, n = tensor.shape
        if not (tensor.stride(0) == 1 and (n <= 1 or tensor.stride(1) >= max(m, 1))):
            raise ValueError("device matrix must be column-major (strides (1, lda))")
        return MatrixHandle(tensor=tensor)

    @property
    def is_sparse(self) -> bool:
        return self._csr is not None

    @property
    def is_device(self) -> bool:
        return self._tensor is not None

    @property
    def nnz(self) -> int:
        return int(self._csr[2].size) if self._csr is not None else self.rows * self.cols

    @property
    def lda(self) -> int:
        if self._tensor is not None:
            return int(self._tensor.stride(1)) if self.cols > 1 else max(self.rows, 1)
        return max(self.rows, 1)

    def to_numpy(self) -> np.ndarray:
        if self._csr is not None:
            rp, ci, v = self._csr
            out = np.zeros((self.rows, self.cols), order="F")
            for i in range(self.rows):
                out[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
            return out
        if self._host is not None:
            return np.array(self._host)
        return self._tensor.detach().cpu().numpy()

    def fro_norm(self) -> float:
        """||A||_F (proj/src/matrix.cpp:297-302); device handles reduce on the device."""
        if self._tensor is not None:
            import torch

            t = self._tensor
            out = C.c_double()
            with torch.cuda.device(t.device):
                stream = torch.cuda.current_stream(t.device).cuda_stream
                _check(_lib().itercur_fro_norm_device(C.c_void_p(t.data_ptr()), self.rows, self.cols, self.lda,
                                                      C.c_void_p(stream), C.byref(out)))
            return out.value
        a = self._host if self._csr is None else np.asfortranarray(self._csr[2].reshape(-1, 1))
        a = np.asfortranarray(a, dtype=np.float64)
        out = C.c_double()
        _check(_lib().itercur_fro_norm_host(a.ctypes.data_as(C.c_void_p), a.shape[0], a.shape[1],
                                            max(a.shape[0], 1), C.byref(out)))
        return out.value

    def __repr__(self) -> str:
        return f"<MatrixHandle {self.rows}x{self.cols} dense{' device' if self.is_device else ''}>"


def _all_finite(a: np.ndarray) -> bool:
    """MatrixHandle's finite check (proj/src/matrix.cpp:73-77) over column panels with torch's
    multi-threaded CPU kernels (no matrix-sized temporary; ~GB/s per core)."""
    if a.size == 0:
        return True
    import torch

    t = torch.from_numpy(a.T if a.flags.f_contiguous else np.ascontiguousarray(a).T)  # (n, m) row-major view
    step = max(1, (1 << 27) // max(a.shape[0], 1))
    return all(bool(torch.isfinite(t[j:j + step]).all()) for j in range(0, t.shape[0], step))


def _as_handle(a) -> MatrixHandle:
    if isinstance(a, MatrixHandle):
        return a._densified_on_device() if a.is_sparse else a
    try:
        import torch

        if isinstance(a, torch.Tensor) and a.is_cuda:
            return MatrixHandle.device(a)
    except ImportError:  # pragma: no cover
        pass
    if hasattr(a, "to_numpy") and hasattr(a, "is_sparse") and not isinstance(a, np.ndarray):
        # a handle of the reference's own binding (module.cpp:36-57: rows / cols / is_sparse /
        # to_numpy): its dense copy is the matrix (CSR handles densify, as to_dense() does)
        return MatrixHandle.dense(a.to_numpy())
    return MatrixHandle.dense(a)


# ------------------------------------------------------------------------- results
class _Run:
    """Owns the C-ABI run handle (device factors) and frees it with the last reference."""

    def __init__(self, ptr, keepalive):
        self.ptr = ptr
        self.keepalive = keepalive

    def __del__(self):
        if self.ptr:
            try:
                _lib().itercur_run_free(self.ptr)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.ptr = None


class CurFactors:
    """C = A(:,J), core = A(I,J)^+, R = A(I,:) (proj/include/itercur/pinv.hpp:57-66;
    Python surface module.cpp:60-68). C, R and core are materialised on demand from the
    device-resident factors."""

    def __init__(self, run: _Run | None, rows, cols):
        self._run = run
        self.row_indices = list(rows)
        self.col_indices = list(cols)

    @property
    def rank(self) -> int:
        return len(self.col_indices)

    def _mat(self, fn, shape):
        out = np.zeros(shape, dtype=np.float64, order="F")
        if self.rank and self._run is not None:
            _check(fn(self._run.ptr, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def c_matrix(self) -> np.ndarray:
        m = _lib().itercur_run_rows(self._run.ptr) if self._run else 0
        return self._mat(_lib().itercur_run_c_matrix, (m, self.rank))

    def r_matrix(self) -> np.ndarray:
        n = _lib().itercur_run_cols(self._run.ptr) if self._run else 0
        return self._mat(_lib().itercur_run_r_matrix, (self.rank, n))

    def core_matrix(self) -> np.ndarray:
        return self._mat(_lib().itercur_run_core_matrix, (self.rank, self.rank))


@dataclass
class IterationRecord:
    """proj/include/itercur/driver.hpp:32-44 (+ per-iteration pivot margins)."""
    k: int
    rho: float
    cols_added: int
    rows_added: int
    col_truncated: bool
    row_truncated: bool
    select_cols_s: float
    row_residual_s: float
    select_rows_s: float
    core_s: float
    downdate_s: float
    min_col_margin: float
    min_row_margin: float


@dataclass
class RunTrace:
    """proj/include/itercur/driver.hpp:46-54 (Python surface module.cpp:70-80)."""
    status: str
    final_rho: float
    threshold: float
    note: str
    iterations: list = field(default_factory=list)
    sketch_s: float = 0.0
    total_s: float = 0.0
    ga_norm: float = 0.0
    steps: list = field(default_factory=list)  # (kind 0=col/1=row, iteration, index, |best|, |second|)
    kernel_launches: int = 0

    @property
    def rhos(self) -> list:
        return [rec.rho for rec in self.iterations]


def _config(epsilon, b, delta, alpha, risk_adjust, max_rank, max_iters, col_method, row_method, pivot_floor, seed,
            sketch, sparse_nnz, profile, row_pivot_floor=None) -> _capi.Config:
    cfg = _capi.Config()
    _lib().itercur_config_default(C.byref(cfg))
    for name, m in (("col_method", col_method), ("row_method", row_method)):
        if m not in _METHODS:  # module.cpp:18-30 parse_method
            raise ValueError(f"unknown selection method '{m}'")
    if sketch not in _SKETCHES:
        raise ValueError(f"unknown sketch kind '{sketch}'")
    cfg.epsilon, cfg.b, cfg.delta, cfg.alpha = float(epsilon), int(b), float(delta), float(alpha)
    cfg.risk_adjust = 1 if risk_adjust else 0
    cfg.max_rank, cfg.max_iters = int(max_rank), int(max_iters)
    cfg.col_method, cfg.row_method = _METHODS[col_method], _METHODS[row_method]
    # module.cpp:95-96 builds both SelectionMethods with the one pivot_floor; the C-ABI keeps one per method
    cfg.pivot_floor, cfg.seed = float(pivot_floor), int(seed)
    cfg.row_pivot_floor = float(pivot_floor if row_pivot_floor is None else row_pivot_floor)
    cfg.sketch_kind, cfg.sparse_nnz = _SKETCHES[sketch], int(sparse_nnz)
    cfg.profile = 1 if profile else 0
    return cfg


def _collect(run_ptr, keepalive):
    L = _lib()
    run = _Run(run_ptr, keepalive)
    r = L.itercur_run_rank(run_ptr)
    I = np.zeros(max(r, 1), dtype=np.int64)
    J = np.zeros(max(r, 1), dtype=np.int64)
    _check(L.itercur_run_indices(run_ptr, I.ctypes.data_as(C.POINTER(C.c_int64)),
                                 J.ctypes.data_as(C.POINTER(C.c_int64))))
    k = L.itercur_run_num_iterations(run_ptr)
    recs = (_capi.IterationRecord * max(k, 1))()
    _check(L.itercur_run_iterations(run_ptr, recs))
    iters = [IterationRecord(int(x.k), x.rho, int(x.cols_added), int(x.rows_added), bool(x.col_truncated),
                             bool(x.row_truncated), x.select_cols_s, x.row_residual_s, x.select_rows_s, x.core_s,
                             x.downdate_s, x.min_col_margin, x.min_row_margin) for x in recs[:k]]
    ns = L.itercur_run_num_steps(run_ptr)
    sk = np.zeros(max(ns, 1), dtype=np.int32)
    si = np.zeros(max(ns, 1), dtype=np.int64)
    sx = np.zeros(max(ns, 1), dtype=np.int64)
    sb = np.zeros(max(ns, 1))
    ss = np.zeros(max(ns, 1))
    _check(L.itercur_run_steps(run_ptr, sk.ctypes.data_as(C.POINTER(C.c_int32)),
                               si.ctypes.data_as(C.POINTER(C.c_int64)), sx.ctypes.data_as(C.POINTER(C.c_int64)),
                               sb.ctypes.data_as(C.POINTER(C.c_double)), ss.ctypes.data_as(C.POINTER(C.c_double))))
    # tolist(): one C loop per array (a Python-level loop over numpy scalars cost ~2.5 ms per
    # config-2 run — 4720 pivot steps — inside every caller's timed region)
    steps = list(zip(sk[:ns].tolist(), si[:ns].tolist(), sx[:ns].tolist(), sb[:ns].tolist(), ss[:ns].tolist()))
    trace = RunTrace(_STATUS[L.itercur_run_status(run_ptr)], L.itercur_run_final_rho(run_ptr),
                     L.itercur_run_threshold(run_ptr), L.itercur_run_note(run_ptr).decode(), iters,
                     L.itercur_run_sketch_seconds(run_ptr), L.itercur_run_total_seconds(run_ptr),
                     L.itercur_run_ga_norm(run_ptr), steps, L.itercur_run_kernel_launches(run_ptr))
    factors = CurFactors(run, I[:r].tolist(), J[:r].tolist())
    return factors, trace


class _ObservedFactors:
    """The factors as they stand after one iteration, handed to an ``observer`` (IterationObserver,
    proj/include/itercur/driver.hpp:70-72). Valid only during the callback: the run continues
    afterwards, so c_matrix / r_matrix / core_matrix raise once it returns."""

    def __init__(self, run_ptr):
        self._ptr = run_ptr
        self.live = True
        L = _lib()
        r = L.itercur_run_rank(run_ptr)
        I = np.zeros(max(r, 1), dtype=np.int64)
        J = np.zeros(max(r, 1), dtype=np.int64)
        _check(L.itercur_run_indices(run_ptr, I.ctypes.data_as(C.POINTER(C.c_int64)),
                                     J.ctypes.data_as(C.POINTER(C.c_int64))))
        self.row_indices = I[:r].tolist()
        self.col_indices = J[:r].tolist()

    @property
    def rank(self) -> int:
        return len(self.col_indices)

    def _mat(self, fn, shape):
        if not self.live:
            raise RuntimeError("observed factors are only valid during the observer callback")
        out = np.zeros(shape, dtype=np.float64, order="F")
        if self.rank:
            _check(fn(self._ptr, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def c_matrix(self):
        return self._mat(_lib().itercur_run_c_matrix, (_lib().itercur_run_rows(self._ptr), self.rank))

    def r_matrix(self):
        return self._mat(_lib().itercur_run_r_matrix, (self.rank, _lib().itercur_run_cols(self._ptr)))

    def core_matrix(self):
        return self._mat(_lib().itercur_run_core_matrix, (self.rank, self.rank))


def _observer_trampoline(observer, errors):
    def cb(_user, run_ptr, rec_ptr):
        snap = None
        try:
            x = C.cast(rec_ptr, C.POINTER(_capi.IterationRecord)).contents
            rec = IterationRecord(int(x.k), x.rho, int(x.cols_added), int(x.rows_added), bool(x.col_truncated),
                                  bool(x.row_truncated), x.select_cols_s, x.row_residual_s, x.select_rows_s,
                                  x.core_s, x.downdate_s, x.min_col_margin, x.min_row_margin)
            snap = _ObservedFactors(run_ptr)
            observer(snap, rec)
            return 0
        except BaseException as e:  # re-raised by iterative_cur after the engine unwinds
            errors.append(e)
            return 1
        finally:
            if snap is not None:
                snap.live = False
    return _capi.OBSERVER_FN(cb)


def iterative_cur(a, epsilon=1e-6, b=50, delta=0.0, alpha=0.05, risk_adjust=False, max_rank=0, max_iters=0,
                  col_method="lupp", row_method="lupp", pivot_floor=1e-13, seed=0, sketch="gaussian",
                  sparse_nnz=8, profile=False, observer=None, row_pivot_floor=None):
    """Run the rank-adaptive decomposition; returns (factors, trace).

    proj/bindings/python/module.cpp:82-103 -> itercur::iterative_cur, proj/src/driver.cpp:48-167.
    Extensions: ``sketch`` / ``sparse_nnz`` (sparse-sign sketch), ``observer(factors, record)``
    called after every iteration (the C++ API's IterationObserver, driver.hpp:70-72; the Python
    binding does not expose it), ``row_pivot_floor`` (the row SelectionMethod's floor; default:
    ``pivot_floor`` for both, as module.cpp:95-96).
    """
    h = _as_handle(a)
    cfg = _config(epsilon, b, delta, alpha, risk_adjust, max_rank, max_iters, col_method, row_method, pivot_floor,
                  seed, sketch, sparse_nnz, profile, row_pivot_floor)
    errors = []
    if observer is not None:
        cb = _observer_trampoline(observer, errors)
        cfg.observer = C.cast(cb, C.c_void_p)
    try:
        return _run(h, cfg)
    except RuntimeError:
        if errors:
            raise errors[0]
        raise


def _run(h, cfg):
    L = _lib()
    out = C.c_void_p()
    if h.is_device:
        import torch

        t = h._tensor
        with torch.cuda.device(t.device):
            stream = torch.cuda.current_stream(t.device).cuda_stream
            _check(L.itercur_iterative_cur_device(C.c_void_p(t.data_ptr()), h.rows, h.cols, h.lda, C.byref(cfg),
                                                  C.c_void_p(stream), C.byref(out)))
        return _collect(out.value, h)
    host = h._host
    _check(L.itercur_iterative_cur_host(host.ctypes.data_as(C.c_void_p), h.rows, h.cols, max(h.rows, 1),
                                        C.byref(cfg), C.byref(out)))
    return _collect(out.value, None)


def slupp_cur(a, rank, seed=0) -> CurFactors:
    """One-shot s-LUPP CUR baseline (proj/src/baselines.cpp:39-62, binding module.cpp:106-108):
    one Gaussian sketch of ceil(1.1 r) rows on stream SluppSketch, r LUPP column pivots, LUPP
    row pivots on A(:, J) — i.e. one block of the engine's iteration with b = r and no
    stopping test. Raises ValueError outside [0, min(m, n)] and RuntimeError("singular cross
    block") as the reference does."""
    h = _as_handle(a)
    r = int(rank)
    if r < 0 or r > min(h.rows, h.cols):
        raise ValueError("rank must lie in [0, min(m, n)]")
    if r == 0:
        return CurFactors(None, [], [])
    cfg = _config(0.0, r, 0.0, 0.05, False, r, 1, "lupp", "lupp", 1e-13, seed, "gaussian", 8, False)
    cfg.sketch_stream = 2
    cfg.sketch_rows = (11 * r + 9) // 10
    factors, _ = _run(h, cfg)
    if factors.rank == 0:
        raise RuntimeError("singular cross block")
    return factors


def true_relative_error(a, factors: CurFactors) -> float:
    """||A - C core R||_F / ||A||_F (proj/src/driver.cpp:169-190) for the GIVEN matrix `a` and the
    run's factors, on the device over column panels (a host `a` is streamed through the device)."""
    h = _as_handle(a)
    if factors.rank == 0 or factors._run is None:
        return 0.0 if h.fro_norm() == 0.0 else 1.0
    out = C.c_double()
    if h.is_device:
        import torch

        t = h._tensor
        with torch.cuda.device(t.device):
            _check(_lib().itercur_true_relative_error_matrix(factors._run.ptr, C.c_void_p(t.data_ptr()), h.rows,
                                                             h.cols, h.lda, 1, C.byref(out)))
    else:
        _check(_lib().itercur_true_relative_error_matrix(factors._run.ptr, h._host.ctypes.data_as(C.c_void_p),
                                                         h.rows, h.cols, max(h.rows, 1), 0, C.byref(out)))
    return out.value


def sketched_relative_error(a, factors: CurFactors, b: int, seed: int = 0, sketch: str = "gaussian",
                            sparse_nnz: int = 8) -> float:
    """make_sketch(seed, b, A) then downdate_col_residual(estimator, factors)
    (proj/src/sketch.cpp:10-41): ||GA - GA(:,J) core R||_F / ||GA||_F for any finished run's
    factors — how run_threshold scores the s-LUPP baseline with the adaptive run's estimator
    (proj/src/bench.cpp:171-174). Raises ValueError for b < 1 or b > m, as make_sketch does."""
    if factors._run is None:
        h = _as_handle(a)
        b = int(b)
        if b < 1:
            raise ValueError("block size must be at least 1")
        if b > h.rows:
            raise ValueError("block exceeds row count")
        return 0.0 if h.fro_norm() == 0.0 else 1.0
    if sketch not in _SKETCHES:
        raise ValueError(f"unknown sketch '{sketch}'")
    out = C.c_double()
    L = _lib()
    if L.itercur_run_holds_matrix(factors._run.ptr):
        _check(L.itercur_sketched_residual_device(factors._run.ptr, int(b), int(seed), _SKETCHES[sketch],
                                                  int(sparse_nnz), C.byref(out)))
        return out.value
    # host-entry run (its device copy of A was released): the given matrix, on the device
    import torch

    h = _as_handle(a)
    t = h._tensor if h.is_device else torch.from_numpy(np.ascontiguousarray(h._host.T)).cuda().t()
    lda = int(t.stride(1)) if t.shape[1] > 1 else max(int(t.shape[0]), 1)
    with torch.cuda.device(t.device):
        _check(L.itercur_sketched_residual_matrix(factors._run.ptr, C.c_void_p(t.data_ptr()), lda, int(b), int(seed),
                                                  _SKETCHES[sketch], int(sparse_nnz), C.byref(out)))
    return out.value


def adjusted_threshold(epsilon, delta, alpha, c) -> float:
    """proj/src/driver.cpp:28-39."""
    out = C.c_double()
    _check(_lib().itercur_adjusted_threshold(float(epsilon), float(delta), float(alpha), int(c), C.byref(out)))
    return out.value


def gratton_tail(c, tau) -> float:
    """proj/src/driver.cpp:41-46."""
    out = C.c_double()
    _check(_lib().itercur_gratton_tail(int(c), float(tau), C.byref(out)))
    return out.value


def preload() -> int:
    """Load every engine kernel on the current CUDA device now instead of on its first launch (CUDA
    lazy module loading), so the first iterative_cur call pays no module loading; returns how many
    kernels were loaded. Done at import when torch has already initialised CUDA."""
    n = C.c_int32(0)
    _check(_lib().itercur_preload(C.byref(n)))
    return n.value


preload_seconds = None  # wall time of the import-time preload (None: not done)


def _preload_at_import():
    global preload_seconds
    try:
        import time

        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            t0 = time.perf_counter()
            preload()
            preload_seconds = time.perf_counter() - t0
    except Exception:  # no device, no CUDA context yet, or the library not built: nothing to do
        pass


def sketch_rows_for_block(b: int) -> int:
    """floor(1.1 b) — proj/include/itercur/sketch.hpp:10."""
    return int(_lib().itercur_sketch_rows_for_block(int(b)))


__all__ = [
    "CurFactors", "IterationRecord", "MatrixHandle", "RunTrace", "__version__", "adjusted_threshold", "slupp_cur",
    "gratton_tail", "iterative_cur", "preload", "sketch_rows_for_block", "sketched_relative_error",
    "true_relative_error",
]

_preload_at_import()

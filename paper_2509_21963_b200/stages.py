"""Stage-level entries of the engine (tests and benchmarks), over CUDA tensors.

Each wraps one C-ABI entry of include/itercur_b200.h:
  gaussian_matrix  -> itercur::gaussian_matrix   (proj/src/rng.cpp:61-67)
  sketch           -> itercur::make_sketch       (proj/src/sketch.cpp:10-24) + sparse-sign
  select_columns / select_rows -> proj/src/select.cpp:121-165 (LUPP)
  time_sketch_kernel -> CUDA-event timing of the DMMA sketch-apply kernel alone
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from ._capi import check as _check

_SKETCHES = {"gaussian": 0, "sparse_sign": 1}


def _stream(t: torch.Tensor):
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _colmajor_ld(t: torch.Tensor) -> int:
    m, n = t.shape
    if t.stride(0) != 1:
        raise ValueError("expected a column-major (strides (1, ld)) tensor")
    return int(t.stride(1)) if n > 1 else max(m, 1)


def colmajor(x, device="cuda") -> torch.Tensor:
    """(m, n) float64 CUDA tensor with column-major strides from a numpy array / tensor."""
    t = torch.as_tensor(np.asarray(x, dtype=np.float64) if not isinstance(x, torch.Tensor) else x)
    t = t.to(device=device, dtype=torch.float64)
    return t.t().contiguous().t()


def gaussian_matrix(rows: int, cols: int, seed: int, stream_tag: int = 1, device="cuda") -> torch.Tensor:
    out = torch.empty(cols, rows, dtype=torch.float64, device=device).t()
    _check(_capi.lib().itercur_gaussian_matrix_device(rows, cols, seed, stream_tag, C.c_void_p(out.data_ptr()),
                                                      _stream(out)))
    return out


def sketch(a: torch.Tensor, b: int, seed: int, kind: str = "gaussian", sparse_nnz: int = 8):
    """(Y (c x n, column-major), ||Y||_F, ||A||_F)."""
    m, n = a.shape
    c = int(_capi.lib().itercur_sketch_rows_for_block(int(b)))
    y = torch.empty(n, max(c, 1), dtype=torch.float64, device=a.device).t()
    ga, an = C.c_double(), C.c_double()
    _check(_capi.lib().itercur_sketch_device(C.c_void_p(a.data_ptr()), m, n, _colmajor_ld(a), int(b), int(seed),
                                             _SKETCHES[kind], int(sparse_nnz), C.c_void_p(y.data_ptr()),
                                             C.byref(ga), C.byref(an), _stream(a)))
    return y[:c], ga.value, an.value


@dataclass
class Selection:
    indices: list
    truncated: bool
    last_pivot_magnitude: float
    best: list
    second: list


def _select(m: torch.Tensor, b: int, is_columns: bool, pivot_floor: float, exclude, method: str = "lupp") -> Selection:
    rows, cols = m.shape
    ex = np.asarray(list(exclude), dtype=np.int64)
    cap = max(int(b), 1) + 1
    idx = np.zeros(cap, dtype=np.int64)
    best = np.zeros(cap)
    second = np.zeros(cap)
    nidx, trunc, last = C.c_int64(), C.c_int32(), C.c_double()
    i64p = C.POINTER(C.c_int64)
    dp = C.POINTER(C.c_double)
    if method not in ("lupp", "qrcp"):
        raise ValueError(f"unknown selection method '{method}'")
    fn = _capi.lib().itercur_select_device if method == "lupp" else _capi.lib().itercur_select_qrcp_device
    _check(fn(
        C.c_void_p(m.data_ptr()), rows, cols, _colmajor_ld(m), int(b), 1 if is_columns else 0, float(pivot_floor),
        ex.ctypes.data_as(i64p), len(ex), idx.ctypes.data_as(i64p), C.byref(nidx), C.byref(trunc), C.byref(last),
        best.ctypes.data_as(dp), second.ctypes.data_as(dp), _stream(m)))
    k = nidx.value
    return Selection([int(v) for v in idx[:k]], bool(trunc.value), last.value, list(best[:k]), list(second[:k]))


def select_columns(m: torch.Tensor, b: int, pivot_floor: float = 1e-13, exclude=(), method="lupp") -> Selection:
    return _select(m, b, True, pivot_floor, exclude, method)


def select_rows(m: torch.Tensor, b: int, pivot_floor: float = 1e-13, exclude=(), method="lupp") -> Selection:
    return _select(m, b, False, pivot_floor, exclude, method)


def time_sketch_kernel(a: torch.Tensor, b: int, kind: str = "gaussian", reps: int = 5):
    """Mean ms per launch of the DMMA sketch-apply kernel alone, plus its launch geometry."""
    m, n = a.shape
    ms = C.c_double()
    ctas, splits, tma = C.c_int32(), C.c_int32(), C.c_int32()
    _check(_capi.lib().itercur_time_sketch_kernel(C.c_void_p(a.data_ptr()), m, n, _colmajor_ld(a), int(b),
                                                  _SKETCHES[kind], int(reps), _stream(a), C.byref(ms),
                                                  C.byref(ctas), C.byref(splits), C.byref(tma)))
    return {"ms": ms.value, "ctas": ctas.value, "splits": splits.value, "tma": bool(tma.value)}


def time_lupp(rows: int, steps: int, reps: int = 10, force_path: int = 0):
    """Mean microseconds per LUPP launch on a random rows x steps W (0 auto, 1 cluster, 2 grid, 3 global,
    4 resident)."""
    us = C.c_double()
    used = C.c_int32()
    _check(_capi.lib().itercur_time_lupp(int(rows), int(steps), int(reps), int(force_path),
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream), C.byref(us),
                                         C.byref(used)))
    return {"us": us.value, "path": used.value}


def time_gemm(M: int, N: int, K: int, reps: int = 10) -> float:
    """Microseconds per launch of the tall-skinny DMMA GEMM (row-residual shape) on random data."""
    us = C.c_double()
    _check(_capi.lib().itercur_time_gemm(int(M), int(N), int(K), int(reps),
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream), C.byref(us)))
    return us.value


def rows_lu_solve(x: torch.Tensor, lu: torch.Tensor) -> torch.Tensor:
    """out(j, :) = D^{-1} x_j for every row j of x (M x w, column-major CUDA), D = Lhat Uhat packed
    in lu (w x w, unit-lower Lhat below the diagonal, Uhat on and above)."""
    M, w = x.shape
    out = torch.zeros(w, M, dtype=torch.float64, device=x.device).t()
    _check(_capi.lib().itercur_rows_lu_solve_device(C.c_void_p(x.data_ptr()), _colmajor_ld(x), M,
                                                    C.c_void_p(lu.data_ptr()), _colmajor_ld(lu), w,
                                                    C.c_void_p(out.data_ptr()), _colmajor_ld(out), _stream(x)))
    return out

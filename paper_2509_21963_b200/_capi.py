"""ctypes binding of include/itercur_b200.h (the engine's C-ABI).

This is exactly the binding a reference-side maintainer would add:
plain pointers and sizes. The library is built in-tree by ``paper_2509_21963_b200.build``;
if it is missing, importing the engine raises — there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ITERCUR_LIB_OVERRIDE") or os.path.join(_HERE, "libitercur_b200.so")  # A/B builds

OK = 0
E_INVALID, E_RANGE, E_DOMAIN, E_RUNTIME, E_LOGIC = 1, 2, 3, 4, 5
E_CUDA, E_OOM = 10, 11

# every symbol declared in include/itercur_b200.h
EXPORTED = [
    "itercur_config_default", "itercur_last_error", "itercur_abi_version",
    "itercur_iterative_cur_device", "itercur_iterative_cur_host",
    "itercur_run_rank", "itercur_run_rows", "itercur_run_cols", "itercur_run_indices", "itercur_run_status",
    "itercur_run_final_rho", "itercur_run_threshold", "itercur_run_sketch_seconds", "itercur_run_total_seconds",
    "itercur_run_ga_norm", "itercur_run_note", "itercur_run_num_iterations", "itercur_run_iterations",
    "itercur_run_kernel_launches", "itercur_run_num_steps", "itercur_run_steps", "itercur_run_c_matrix", "itercur_run_r_matrix",
    "itercur_run_core_matrix", "itercur_true_relative_error_device", "itercur_sketched_residual_device", "itercur_fro_norm_device",
    "itercur_run_free",
    "itercur_adjusted_threshold", "itercur_gratton_tail", "itercur_sketch_rows_for_block",
    "itercur_gaussian_matrix_device", "itercur_sketch_device", "itercur_select_device",
    "itercur_time_sketch_kernel", "itercur_time_lupp", "itercur_time_gemm",
    "itercur_lupp_dist_step", "itercur_gemm_device", "itercur_block_lu_device", "itercur_rows_lu_solve_device",
    "itercur_select_qrcp_device", "itercur_csr_to_dense_device",
    "itercur_true_relative_error_matrix", "itercur_run_core_apply", "itercur_sketched_residual_matrix",
    "itercur_run_holds_matrix", "itercur_copy_to_host",
    "itercur_shard_range", "itercur_iterative_cur_sharded_device", "itercur_iterative_cur_sharded_emulated",
    "itercur_true_relative_error_sharded", "itercur_nccl_unique_id", "itercur_nccl_comm_init",
    "itercur_nccl_comm_destroy", "itercur_fro_norm_host", "itercur_dense_apply_host", "itercur_preload",
]


class Config(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double), ("b", C.c_int64), ("delta", C.c_double), ("alpha", C.c_double),
        ("risk_adjust", C.c_int32), ("max_rank", C.c_int64), ("max_iters", C.c_int64),
        ("col_method", C.c_int32), ("row_method", C.c_int32), ("pivot_floor", C.c_double),
        ("seed", C.c_uint64), ("sketch_kind", C.c_int32), ("sparse_nnz", C.c_int32),
        ("profile", C.c_int32), ("sketch_stream", C.c_int32), ("sketch_rows", C.c_int64),
        ("row_pivot_floor", C.c_double), ("observer", C.c_void_p), ("observer_user", C.c_void_p),
        ("keep_device_copy", C.c_int32),
    ]


# int (*)(void* user, const itercur_run* run, const itercur_iteration_record* record)
OBSERVER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class IterationRecord(C.Structure):
    _fields_ = [
        ("k", C.c_int64), ("rho", C.c_double), ("cols_added", C.c_int64), ("rows_added", C.c_int64),
        ("col_truncated", C.c_int32), ("row_truncated", C.c_int32), ("select_cols_s", C.c_double),
        ("row_residual_s", C.c_double), ("select_rows_s", C.c_double), ("core_s", C.c_double),
        ("downdate_s", C.c_double), ("min_col_margin", C.c_double), ("min_row_margin", C.c_double),
    ]


_lib = None


def lib() -> C.CDLL:
    """Load libitercur_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2509_21963_b200.build` "
                          "(the B200 engine has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, dp, i64p, i32p = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    runp = C.c_void_p
    sig = {
        "itercur_config_default": (None, [C.POINTER(Config)]),
        "itercur_last_error": (C.c_char_p, []),
        "itercur_abi_version": (C.c_int, []),
        "itercur_preload": (C.c_int, [C.POINTER(C.c_int32)]),
        "itercur_iterative_cur_device": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.POINTER(Config), vp,
                                                   C.POINTER(runp)]),
        "itercur_iterative_cur_host": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.POINTER(Config),
                                                 C.POINTER(runp)]),
        "itercur_run_rank": (C.c_int64, [runp]),
        "itercur_run_rows": (C.c_int64, [runp]),
        "itercur_run_cols": (C.c_int64, [runp]),
        "itercur_run_indices": (C.c_int, [runp, i64p, i64p]),
        "itercur_run_status": (C.c_int32, [runp]),
        "itercur_run_final_rho": (C.c_double, [runp]),
        "itercur_run_threshold": (C.c_double, [runp]),
        "itercur_run_sketch_seconds": (C.c_double, [runp]),
        "itercur_run_total_seconds": (C.c_double, [runp]),
        "itercur_run_ga_norm": (C.c_double, [runp]),
        "itercur_run_note": (C.c_char_p, [runp]),
        "itercur_run_num_iterations": (C.c_int64, [runp]),
        "itercur_run_iterations": (C.c_int, [runp, C.POINTER(IterationRecord)]),
        "itercur_run_num_steps": (C.c_int64, [runp]),
        "itercur_run_kernel_launches": (C.c_int64, [runp]),
        "itercur_run_steps": (C.c_int, [runp, i32p, i64p, i64p, dp, dp]),
        "itercur_run_c_matrix": (C.c_int, [runp, dp]),
        "itercur_run_r_matrix": (C.c_int, [runp, dp]),
        "itercur_run_core_matrix": (C.c_int, [runp, dp]),
        "itercur_true_relative_error_device": (C.c_int, [runp, dp]),
        "itercur_true_relative_error_matrix": (C.c_int, [runp, vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32, dp]),
        "itercur_run_core_apply": (C.c_int, [runp, C.c_int32, vp, C.c_int64, C.c_int64, vp, C.c_int64]),
        "itercur_sketched_residual_matrix": (C.c_int, [runp, vp, C.c_int64, C.c_int64, C.c_uint64, C.c_int32,
                                                       C.c_int32, dp]),
        "itercur_run_holds_matrix": (C.c_int32, [runp]),
        "itercur_copy_to_host": (C.c_int, [vp, vp, C.c_uint64]),
        "itercur_shard_range": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, i64p, i64p]),
        "itercur_iterative_cur_sharded_device": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                                           C.POINTER(Config), vp, vp, C.POINTER(runp)]),
        "itercur_iterative_cur_sharded_emulated": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                                             C.POINTER(Config), vp, C.POINTER(runp)]),
        "itercur_true_relative_error_sharded": (C.c_int, [runp, dp]),
        "itercur_nccl_unique_id": (C.c_int, [vp]),
        "itercur_nccl_comm_init": (C.c_int, [C.c_int32, vp, C.c_int32, C.POINTER(vp)]),
        "itercur_nccl_comm_destroy": (C.c_int, [vp]),
        "itercur_fro_norm_host": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, dp]),
        "itercur_dense_apply_host": (C.c_int, [vp, C.c_int64, C.c_int32, vp, C.c_int64, vp]),
        "itercur_fro_norm_device": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, vp, dp]),
        "itercur_sketched_residual_device": (C.c_int, [runp, C.c_int64, C.c_uint64, C.c_int32, C.c_int32, dp]),
        "itercur_run_free": (None, [runp]),
        "itercur_adjusted_threshold": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int64, dp]),
        "itercur_gratton_tail": (C.c_int, [C.c_int64, C.c_double, dp]),
        "itercur_sketch_rows_for_block": (C.c_int64, [C.c_int64]),
        "itercur_gaussian_matrix_device": (C.c_int, [C.c_int64, C.c_int64, C.c_uint64, C.c_uint32, vp, vp]),
        "itercur_sketch_device": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int32,
                                            C.c_int32, vp, dp, dp, vp]),
        "itercur_select_device": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_double,
                                            i64p, C.c_int64, i64p, i64p, i32p, dp, dp, dp, vp]),
        "itercur_csr_to_dense_device": (C.c_int, [C.c_int64, C.c_int64, vp, vp, vp, vp, C.c_int64, vp]),
        "itercur_select_qrcp_device": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                                 C.c_double, i64p, C.c_int64, i64p, i64p, i32p, dp, dp, dp, vp]),
        "itercur_time_sketch_kernel": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                                 C.c_int32, vp, dp, i32p, i32p, i32p]),
        "itercur_time_lupp": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_int32, vp, dp, i32p]),
        "itercur_time_gemm": (C.c_int, [C.c_int64, C.c_int32, C.c_int64, C.c_int32, vp, dp]),
        "itercur_lupp_dist_step": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int32, C.c_int32, vp, C.c_int64, vp,
                                             C.c_int64, vp, vp]),
        "itercur_gemm_device": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, vp, C.c_int64, vp, C.c_int64, vp,
                                          C.c_int64, C.c_double, vp, C.c_int64, vp]),
        "itercur_block_lu_device": (C.c_int, [vp, C.c_int64, C.c_int64, vp]),
        "itercur_rows_lu_solve_device": (C.c_int, [vp, C.c_int64, C.c_int64, vp, C.c_int64, C.c_int64, vp, C.c_int64,
                                                   vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


_EXC = {E_INVALID: ValueError, E_RANGE: IndexError, E_DOMAIN: ValueError, E_RUNTIME: RuntimeError,
        E_LOGIC: RuntimeError, E_CUDA: RuntimeError, E_OOM: MemoryError}


def check(rc: int) -> None:
    """Map a C-ABI status to the exception class pybind11 gives the reference's C++ one."""
    if rc != OK:
        msg = lib().itercur_last_error().decode(errors="replace")
        raise _EXC.get(rc, RuntimeError)(msg)

/*
 * itercur_b200.h — C-ABI of the B200-native IterativeCUR engine (drop-in boundary).
 *
 * Plain pointers and sizes only (no torch / Eigen types). Each entry point replaces one
 * reference interface (paths relative to /root/reference):
 *
 *   itercur_iterative_cur_host / _device
 *       itercur::iterative_cur            proj/include/itercur/driver.hpp:79-81
 *                                         (body proj/src/driver.cpp:48-167)
 *       and the pybind11 binding          proj/bindings/python/module.cpp:82-103
 *   itercur_config (+ itercur_config_default)
 *       itercur::StoppingConfig           proj/include/itercur/driver.hpp:18-26
 *       itercur::SelectionMethod          proj/include/itercur/select.hpp:12-15
 *   itercur_run_* accessors
 *       itercur::CurFactors               proj/include/itercur/pinv.hpp:57-66
 *       itercur::RunTrace / IterationRecord  proj/include/itercur/driver.hpp:32-54
 *       CurFactors.c_matrix/r_matrix/core_matrix  proj/bindings/python/module.cpp:60-68
 *   itercur_true_relative_error_device
 *       itercur::true_relative_error      proj/include/itercur/driver.hpp:85 (driver.cpp:169-190)
 *   itercur_sketched_residual_device
 *       make_sketch + downdate_col_residual  proj/src/sketch.cpp:10-41 (as run_threshold, bench.cpp:171-174)
 *   itercur_adjusted_threshold / itercur_gratton_tail
 *       proj/include/itercur/driver.hpp:64,68 (driver.cpp:28-46)
 *   itercur_sketch_device
 *       itercur::make_sketch              proj/include/itercur/sketch.hpp:36 (sketch.cpp:10-24)
 *   itercur_select_device
 *       itercur::select_columns / select_rows  proj/include/itercur/select.hpp:31-38
 *   itercur_gaussian_matrix_device
 *       itercur::gaussian_matrix          proj/include/itercur/rng.hpp:33-34 (rng.cpp:61-67)
 *
 * Matrices are column-major doubles (the reference's Eigen default). Indices are int64
 * (itercur::Index, proj/include/itercur/matrix.hpp:12).
 *
 * Errors: every entry returns ITERCUR_OK or a code naming the reference's exception class
 * (std::invalid_argument, out_of_range, domain_error, runtime_error, logic_error), or a
 * CUDA failure; itercur_last_error() returns the message (thread-local), preserving the
 * reference's texts ("matrix must be nonzero", "block exceeds row count", "block too
 * small for requested alpha", "not implemented", ...). Non-exceptional ends are reported
 * through the run status, as in the reference.
 *
 * There is no CPU fallback: without a usable sm_100 device every compute entry returns
 * ITERCUR_E_CUDA.
 */
#ifndef ITERCUR_B200_H
#define ITERCUR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ITERCUR_B200_ABI_VERSION 4

#if defined(__GNUC__)
#define ITERCUR_API __attribute__((visibility("default")))
#else
#define ITERCUR_API
#endif

enum itercur_status_code {
  ITERCUR_OK = 0,
  ITERCUR_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  ITERCUR_E_OUT_OF_RANGE = 2,     /* std::out_of_range */
  ITERCUR_E_DOMAIN = 3,           /* std::domain_error */
  ITERCUR_E_RUNTIME = 4,          /* std::runtime_error */
  ITERCUR_E_LOGIC = 5,            /* std::logic_error */
  ITERCUR_E_CUDA = 10,            /* CUDA launch / runtime failure */
  ITERCUR_E_OOM = 11              /* device allocation failed */
};

enum itercur_run_status { ITERCUR_CONVERGED = 0, ITERCUR_MAX_RANK = 1, ITERCUR_RESIDUAL_EXHAUSTED = 2 };
enum itercur_pivot_kind { ITERCUR_PIVOT_LUPP = 0, ITERCUR_PIVOT_QRCP = 1, ITERCUR_PIVOT_OSINSKY = 2 };
enum itercur_sketch_kind { ITERCUR_SKETCH_GAUSSIAN = 0, ITERCUR_SKETCH_SPARSE_SIGN = 1 };

struct itercur_run;
struct itercur_iteration_record;
/* IterationObserver (proj/include/itercur/driver.hpp:70-72, called at driver.cpp:154): invoked after
   each completed iteration with the run as it stands (rank, indices, factors through the
   itercur_run_* accessors) and that iteration's record. A nonzero return aborts the run with
   ITERCUR_E_RUNTIME ("iteration observer failed"). With an observer the engine runs one iteration
   per device batch (slow path; the reference uses it in tests). */
typedef int (*itercur_observer_fn)(void* user, const struct itercur_run* run,
                                   const struct itercur_iteration_record* record);

/* StoppingConfig + the two SelectionMethods + seed + the new sketch options. */
typedef struct itercur_config {
  double epsilon;      /* 1e-6  */
  int64_t b;           /* 50    */
  double delta;        /* 0.0   */
  double alpha;        /* 0.05  */
  int32_t risk_adjust; /* 0     */
  int64_t max_rank;    /* 0 -> min(m, n) */
  int64_t max_iters;   /* 0 -> ceil(min(m, n) / b) + 1 */
  int32_t col_method;  /* ITERCUR_PIVOT_LUPP */
  int32_t row_method;  /* ITERCUR_PIVOT_LUPP */
  double pivot_floor;  /* 1e-13: col_method.pivot_floor (select.hpp:12-15) */
  uint64_t seed;       /* 0 */
  int32_t sketch_kind; /* ITERCUR_SKETCH_GAUSSIAN (the reference's only kind) */
  int32_t sparse_nnz;  /* 8 */
  int32_t profile;     /* 1: record per-phase CUDA-event times into the trace */
  int32_t sketch_stream; /* 0 -> RngStream::Sketch (1); 2 = SluppSketch (the s-LUPP baseline) */
  int64_t sketch_rows;   /* 0 -> floor(1.1 b) (sketch.hpp:10); > 0 overrides (s-LUPP: ceil(1.1 r)) */
  /* ABI 4 */
  double row_pivot_floor;        /* 1e-13: row_method.pivot_floor; <= 0 -> pivot_floor */
  itercur_observer_fn observer;  /* NULL: none */
  void* observer_user;           /* passed back to observer */
  int32_t keep_device_copy;      /* host entry: 1 keeps the device copy of A alive with the run (the
                                    accessors and the run-matrix error / sketched residual then use it);
                                    0 (default) frees it when the call returns, keeping only compact
                                    gathers of C = A(:,J) and R = A(I,:) */
} itercur_config;

/* One IterationRecord (proj/include/itercur/driver.hpp:32-44) plus pivot-margin data. */
typedef struct itercur_iteration_record {
  int64_t k;
  double rho;
  int64_t cols_added;
  int64_t rows_added;
  int32_t col_truncated;
  int32_t row_truncated;
  double select_cols_s;
  double row_residual_s;
  double select_rows_s;
  double core_s;
  double downdate_s;
  double min_col_margin; /* min over steps of (|best|-|second|)/|best| in the column LUPP */
  double min_row_margin; /* same for the row LUPP */
} itercur_iteration_record;

typedef struct itercur_run itercur_run; /* opaque: CurFactors + RunTrace + device buffers */

ITERCUR_API void itercur_config_default(itercur_config* cfg);
ITERCUR_API const char* itercur_last_error(void);
ITERCUR_API int itercur_abi_version(void);

/* iterative_cur on a device-resident column-major A (m x n, leading dimension lda).
   `stream` is a cudaStream_t (NULL = legacy default stream). A must stay alive and
   unmodified while the run handle is used for c/r/core/error queries. */
ITERCUR_API int itercur_iterative_cur_device(const double* dA, int64_t m, int64_t n, int64_t lda, const itercur_config* cfg,
                                 void* stream, itercur_run** out);
/* Same, from a host buffer: A is copied to the current device inside the call (the copy
   is part of the call, as in the reference binding's numpy -> Eigen copy). The run keeps
   the device copy alive until itercur_run_free. */
ITERCUR_API int itercur_iterative_cur_host(const double* A, int64_t m, int64_t n, int64_t lda, const itercur_config* cfg,
                               itercur_run** out);

/* ---- column-sharded runs (one process per GPU over NCCL) ----
 * A is split by columns into contiguous blocks: rank r of `world` owns columns
 * [off, off + count) from itercur_shard_range (blocks of an even width). Each rank passes its block
 * (m x count, ld lda, on its device) and a ncclComm_t over the ranks; every rank returns the same
 * indices, status and trace as one device would (the sketch is local, the column selection runs on
 * the replicated Y^T(:, 0:b), gathered per iteration; the selected block [A(:,J_k) | R~(:,J_k) |
 * Y(:,J_k)] is assembled with one sum-allreduce of disjoint contributions; ||Y||^2 with one scalar
 * allreduce; the row selection, L and D_k are replicated; the U block and the downdate are local).
 * All collectives are enqueued on the run's stream and captured in its iteration graphs. A rank
 * holds only its columns of A, Y and R~: C / R / core exports are not available on it (indices,
 * trace and itercur_true_relative_error_sharded are). NCCL (libnccl.so.2) is loaded at run time. */
ITERCUR_API int itercur_shard_range(int64_t n_total, int32_t world, int32_t rank, int64_t* offset, int64_t* count);
ITERCUR_API int itercur_iterative_cur_sharded_device(const double* dA, int64_t m, int64_t n_local, int64_t lda,
                                                     int64_t n_total, const itercur_config* cfg, void* nccl_comm,
                                                     void* stream, itercur_run** out);
/* The same pipeline with `shards` column shards computed by ONE process on its device (per-shard
 * kernels on each shard's columns; the collectives become the equivalent device writes): the
 * multi-rank data path exercised on one GPU. dA is the whole m x n matrix. */
ITERCUR_API int itercur_iterative_cur_sharded_emulated(const double* dA, int64_t m, int64_t n, int64_t lda,
                                                       int32_t shards, const itercur_config* cfg, void* stream,
                                                       itercur_run** out);
/* true_relative_error over a sharded run: collective on the run's communicator (every rank calls it). */
ITERCUR_API int itercur_true_relative_error_sharded(const itercur_run* run, double* out);
/* NCCL plumbing for callers without their own communicator: the 128-byte unique id (rank 0; share
 * it with the other ranks), the communicator on the current device, and its release. */
ITERCUR_API int itercur_nccl_unique_id(void* id_out);
ITERCUR_API int itercur_nccl_comm_init(int32_t world, const void* id, int32_t rank, void** comm_out);
ITERCUR_API int itercur_nccl_comm_destroy(void* comm);

/* ---- run accessors (CurFactors / RunTrace) ---- */
ITERCUR_API int64_t itercur_run_rank(const itercur_run* run);
ITERCUR_API int64_t itercur_run_rows(const itercur_run* run);
ITERCUR_API int64_t itercur_run_cols(const itercur_run* run);
ITERCUR_API int itercur_run_indices(const itercur_run* run, int64_t* row_indices, int64_t* col_indices);
ITERCUR_API int32_t itercur_run_status(const itercur_run* run);
ITERCUR_API double itercur_run_final_rho(const itercur_run* run);
ITERCUR_API double itercur_run_threshold(const itercur_run* run);
ITERCUR_API double itercur_run_sketch_seconds(const itercur_run* run);
ITERCUR_API double itercur_run_total_seconds(const itercur_run* run);
ITERCUR_API double itercur_run_ga_norm(const itercur_run* run);
ITERCUR_API const char* itercur_run_note(const itercur_run* run);
ITERCUR_API int64_t itercur_run_num_iterations(const itercur_run* run);
ITERCUR_API int itercur_run_iterations(const itercur_run* run, itercur_iteration_record* out);
/* number of this library's kernels the run launched (sketch + iterations) */
ITERCUR_API int64_t itercur_run_kernel_launches(const itercur_run* run);
/* per pivot step log: kind (0 col, 1 row), iteration, index, |best|, |second| */
ITERCUR_API int64_t itercur_run_num_steps(const itercur_run* run);
ITERCUR_API int itercur_run_steps(const itercur_run* run, int32_t* kind, int64_t* iter, int64_t* index, double* best,
                      double* second);
/* C = A(:, J) (m x r), R = A(I, :) (r x n), core = A(I, J)^{-1} (r x r); host outputs,
   column-major. core is materialised from the engine's block-LU factors on demand
   (FactoredPinv::materialize, proj/src/pinv.cpp:40-43). */
ITERCUR_API int itercur_run_c_matrix(const itercur_run* run, double* out);
ITERCUR_API int itercur_run_r_matrix(const itercur_run* run, double* out);
ITERCUR_API int itercur_run_core_matrix(const itercur_run* run, double* out);
/* ||A - CUR||_F / ||A||_F evaluated on the device over column panels. */
ITERCUR_API int itercur_true_relative_error_device(const itercur_run* run, double* out);
/* true_relative_error(A, factors) (proj/src/driver.cpp:169-190) for a GIVEN matrix A (m x n, the
   run's shape; ld lda) and the run's factors: ||A - C core R||_F / ||A||_F. a_on_device = 1: dA is a
   device pointer; 0: a host buffer streamed to the device in column panels. */
ITERCUR_API int itercur_true_relative_error_matrix(const itercur_run* run, const double* A, int64_t m, int64_t n,
                                                   int64_t lda, int32_t a_on_device, double* out);
/* FactoredPinv::solve / solve_transposed (proj/include/itercur/pinv.hpp:27-33) of the run's core:
   out = X^{-1} rhs (transposed = 0) or X^{-T} rhs (1), X = A(I, J) (r x r), rhs r x k (ld ldr),
   out r x k (ld ldo); host buffers, computed on the device from the block-LU factors. */
ITERCUR_API int itercur_run_core_apply(const itercur_run* run, int32_t transposed, const double* rhs, int64_t k,
                                       int64_t ldr, double* out, int64_t ldo);
/* make_sketch(seed, b, A) then downdate_col_residual(estimator, factors) for the run's factors
 * (proj/src/sketch.cpp:10-41; used by run_threshold, proj/src/bench.cpp:171-174, to score the
 * s-LUPP baseline with the adaptive run's estimator): out = ||GA - GA(:,J) X^{-1} R||_F / ||GA||_F. */
/* The same for a given device matrix dA (the run's shape, ld lda) — for host-entry runs that no
   longer hold A. */
ITERCUR_API int itercur_sketched_residual_matrix(const itercur_run* run, const double* dA, int64_t lda, int64_t b,
                                                 uint64_t seed, int32_t kind, int32_t sparse_nnz, double* out);
/* 1 when the run still references a device copy of its input (device entry, or host entry with
   keep_device_copy), else 0. */
ITERCUR_API int32_t itercur_run_holds_matrix(const itercur_run* run);
/* Copy `bytes` from device memory to host memory on the current device (plumbing for bindings
   that do not link the CUDA runtime themselves, e.g. the C++ facade's MatrixHandle::device). */
ITERCUR_API int itercur_copy_to_host(void* dst, const void* d_src, uint64_t bytes);
/* ||A||_F of a device matrix (proj/src/matrix.cpp:297-302 fro_norm), fixed-order reduction. */
ITERCUR_API int itercur_fro_norm_device(const double* dA, int64_t m, int64_t n, int64_t lda, void* stream, double* out);
/* The same for a host matrix (streamed through the device in column panels). */
ITERCUR_API int itercur_fro_norm_host(const double* A, int64_t m, int64_t n, int64_t lda, double* out);
/* out = X * rhs (transposed = 0) or X^T * rhs (1) for a host r x r matrix X and r x k rhs (column-major,
   ld r / r / r), computed on the device GEMM: the C++ facade's FactoredPinv for observer snapshots,
   which hold the materialised core (no host arithmetic in the bindings). */
ITERCUR_API int itercur_dense_apply_host(const double* X, int64_t r, int32_t transposed, const double* rhs, int64_t k,
                                         double* out);
ITERCUR_API int itercur_sketched_residual_device(const itercur_run* run, int64_t b, uint64_t seed, int32_t kind,
                                                 int32_t sparse_nnz, double* out);
ITERCUR_API void itercur_run_free(itercur_run* run);

/* ---- helpers ---- */
ITERCUR_API int itercur_adjusted_threshold(double epsilon, double delta, double alpha, int64_t c, double* out);
ITERCUR_API int itercur_gratton_tail(int64_t c, double tau, double* out);
ITERCUR_API int64_t itercur_sketch_rows_for_block(int64_t b);

/* ---- stage-level entries (tests / benchmarks) ---- */
/* G (rows x cols, column-major, device) with G(i, j) = normal_at(seed, stream, i, j). */
ITERCUR_API int itercur_gaussian_matrix_device(int64_t rows, int64_t cols, uint64_t seed, uint32_t stream_tag, double* dOut,
                                   void* stream);
/* Y = S * A (c x n, ld c), ||Y||_F and ||A||_F; S Gaussian or sparse-sign. */
ITERCUR_API int itercur_sketch_device(const double* dA, int64_t m, int64_t n, int64_t lda, int64_t b, uint64_t seed,
                          int32_t kind, int32_t sparse_nnz, double* dY, double* ga_norm, double* a_norm, void* stream);
/* LUPP selection on a device matrix M (rows x cols, ld): is_columns = 1 -> select_columns(M, b),
   0 -> select_rows(M, b). Host outputs (idx capacity >= b). */
ITERCUR_API int itercur_select_device(const double* dM, int64_t rows, int64_t cols, int64_t ldm, int64_t b, int32_t is_columns,
                          double pivot_floor, const int64_t* exclude, int64_t n_exclude, int64_t* idx_out,
                          int64_t* n_idx, int32_t* truncated, double* last_pivot, double* best_out,
                          double* second_out, void* stream);
/* Time the sketch-apply DMMA kernel alone (CUDA events on `stream`), `reps` launches;
   returns the mean milliseconds per launch and the kernel's launch geometry. */
/* The same selections by QRCP (greedy orthogonalised column norms, select.cpp:79-117):
 * candidates are the columns of M (is_columns=1, select.cpp:121-139) or its rows
 * (select.cpp:141-165); second_out entries are -1 (no runner-up is tracked). */
ITERCUR_API int itercur_select_qrcp_device(const double* dM, int64_t rows, int64_t cols, int64_t ldm, int64_t b,
                                           int32_t is_columns, double pivot_floor, const int64_t* exclude,
                                           int64_t n_exclude, int64_t* idx_out, int64_t* n_idx, int32_t* truncated,
                                           double* last_pivot, double* best_out, double* second_out, void* stream);
ITERCUR_API int itercur_time_sketch_kernel(const double* dA, int64_t m, int64_t n, int64_t lda, int64_t b, int32_t kind,
                               int32_t reps, void* stream, double* ms_per_launch, int32_t* ctas, int32_t* splits,
                               int32_t* uses_tma);

/* Time the LUPP selection kernel alone on a random rows x steps column-major W (CUDA
   events, `reps` launches after one warm-up). path_used: -CL for the cluster kernel,
   G for the grid shared-memory kernel, 1000000 + G for the global-memory kernel. */
ITERCUR_API int itercur_time_lupp(int64_t rows, int32_t steps, int32_t reps, int32_t force_path, void* stream,
                                  double* us_per_launch, int32_t* path_used);

/* Time the tall-skinny DMMA GEMM C = A(:,idx) - L * B (the row-residual shape) on random
   data: M x K times K x N, `reps` launches; returns microseconds per launch. */
/* CSR input (MatrixHandle sparse path, proj/src/matrix.cpp:79-104): scatter a validated CSR
 * matrix (int64 row_ptr / col_idx, double values, all device pointers) into a dense column-major
 * rows x cols buffer (ld >= rows) that the dense entries then take. */
ITERCUR_API int itercur_csr_to_dense_device(int64_t rows, int64_t cols, const int64_t* dRowPtr, const int64_t* dColIdx,
                                            const double* dValues, double* dOut, int64_t ld, void* stream);

/* ---- column-sharded engine building blocks (paper_2509_21963_b200/sharded.py) ----
 * One pivot step of the distributed column LUPP on this rank's rows of W = Y^T (select.cpp:34-74):
 * eliminate the live rows with the previous step's pivot row dPivotRow (NULL at s == 0; the pivot's
 * local row, if owned, is retired first), then write this rank's candidate for column s to dCand:
 * [|best| (-1 if none), runner-up, global row index, 0, row tail W(best, 0..steps-1) (entries < s are 0)]. */
ITERCUR_API int itercur_lupp_dist_step(double* dW, int64_t rows, int64_t ldw, int32_t steps, int32_t s,
                                       const double* dPivotRow, int64_t pivot_local_row, uint8_t* dLive,
                                       int64_t row_offset, double* dCand, void* stream);
/* C(:, q) = base(:, q) + alpha * A * B(:, q), column-major (M x K, K x N), on the engine's DMMA GEMM
 * (row residual sketch.cpp:56-58 / U block pinv.cpp:94-111 shapes). dBase may be NULL (base = 0);
 * lda must be even and dA 16-byte aligned. */
ITERCUR_API int itercur_gemm_device(int64_t M, int64_t N, int64_t K, const double* dA, int64_t lda, const double* dB,
                                    int64_t ldb, const double* dBase, int64_t ldbase, double alpha, double* dC,
                                    int64_t ldc, void* stream);
/* In-place LU without pivoting of the w x w cross block (rows already in LUPP order). */
ITERCUR_API int itercur_block_lu_device(double* dD, int64_t w, int64_t ldd, void* stream);
/* out(j, :) = D^{-1} x_j for every row j of X (M x w): forward then back substitution with the
 * factors of itercur_block_lu_device (never an explicit inverse). */
ITERCUR_API int itercur_rows_lu_solve_device(const double* dX, int64_t ldx, int64_t M, const double* dLU, int64_t ldd,
                                             int64_t w, double* dOut, int64_t ldo, void* stream);

ITERCUR_API int itercur_time_gemm(int64_t M, int32_t N, int64_t K, int32_t reps, void* stream, double* us_per_launch);

/* Load every engine kernel now instead of on its first launch (CUDA lazy module loading): the first
 * iterative_cur call in a process then pays no module loading. Called by the Python package at import
 * when a CUDA device is present. functions_loaded (optional): how many kernels were loaded. */
ITERCUR_API int itercur_preload(int32_t* functions_loaded);

#ifdef __cplusplus
}
#endif
#endif /* ITERCUR_B200_H */

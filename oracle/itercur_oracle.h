/*
 * itercur_oracle.h — C API of the CPU ORACLE (test infrastructure, NOT the product).
 *
 * A plain-C++ restatement of the reference IterativeCUR hot path
 * (/root/reference/proj/src/{rng,sketch,select,pinv,matrix,driver}.cpp) used only
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg, always as the checker or the timed CPU baseline — never as the product path.
 *
 * Pinning: the Philox / normal / uniform stream is pinned bit-for-bit against the
 * reference's own proj/src/rng.cpp (compiled into oracle/_ref by oracle/Makefile;
 * vectors committed under tests/golden/). The LUPP, sketch, driver and core
 * semantics are pinned by restating the reference's own unit tests
 * (proj/tests/test_{select,sketch,driver,pinv}.cpp) in tests/test_oracle_*.py.
 * The sparse-sign stream has no reference implementation: it is
 * defined here — parity for that variant is "unpinned" w.r.t.
 * the reference and pinned only by this oracle's own known-answer vectors.
 *
 * Error convention (mirrors the reference's exception classes):
 * every entry returns 0 on success or one of ORACLE_E_* and leaves a message in
 * oracle_last_error().
 */
#ifndef ITERCUR_ORACLE_H
#define ITERCUR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORACLE_OK = 0,
  ORACLE_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  ORACLE_E_OUT_OF_RANGE = 2,     /* std::out_of_range */
  ORACLE_E_DOMAIN = 3,           /* std::domain_error */
  ORACLE_E_RUNTIME = 4,          /* std::runtime_error */
  ORACLE_E_LOGIC = 5             /* std::logic_error */
};

/* proj/include/itercur/rng.hpp:12-19 stream tags, plus the new SparseSign = 7. */
enum { ORACLE_STREAM_SKETCH = 1, ORACLE_STREAM_SLUPP_SKETCH = 2, ORACLE_STREAM_SPARSE_SIGN = 7 };
enum { ORACLE_SKETCH_GAUSSIAN = 0, ORACLE_SKETCH_SPARSE_SIGN = 1 };
enum { ORACLE_PIVOT_LUPP = 0, ORACLE_PIVOT_QRCP = 1, ORACLE_PIVOT_OSINSKY = 2 };
enum { ORACLE_CONVERGED = 0, ORACLE_MAX_RANK = 1, ORACLE_RESIDUAL_EXHAUSTED = 2 };

typedef struct {
  double epsilon;      /* StoppingConfig, proj/include/itercur/driver.hpp:18-26 */
  int64_t b;
  double delta;
  double alpha;
  int32_t risk_adjust;
  int64_t max_rank;
  int64_t max_iters;
  int32_t col_method;  /* SelectionMethod, proj/include/itercur/select.hpp:12-15 */
  int32_t row_method;
  double pivot_floor;
  uint64_t seed;
  int32_t sketch_kind; /* new: 0 Gaussian (reference), 1 sparse-sign */
  int32_t sparse_nnz;  /* new: nonzeros per column of the sparse-sign embedding (8) */
} oracle_config;

typedef struct {
  /* caller-provided buffers and their capacities */
  int64_t cap_rank;        /* capacity of row_indices / col_indices */
  int64_t* row_indices;    /* I */
  int64_t* col_indices;    /* J */
  int64_t cap_iters;       /* capacity of the per-iteration arrays */
  double* rhos;            /* rho after each iteration */
  int64_t* widths;         /* cols_added (= rows_added) per iteration */
  double* iter_seconds;    /* wall seconds of each iteration (may be NULL) */
  int64_t cap_steps;       /* capacity of the per-pivot-step log (may be 0) */
  int32_t* step_kind;      /* 0 column LUPP, 1 row LUPP */
  int64_t* step_iter;      /* iteration k */
  int64_t* step_index;     /* chosen pivot */
  double* step_best;       /* |best| */
  double* step_second;     /* |second best| among unbanned candidates (-1 if none) */
  /* outputs */
  int64_t rank;
  int64_t n_iters;
  int64_t n_steps;         /* steps logged (may exceed cap_steps; only cap_steps stored) */
  int32_t status;          /* ORACLE_CONVERGED / MAX_RANK / RESIDUAL_EXHAUSTED */
  double final_rho;
  double threshold;
  double sketch_s;
  double total_s;
  double ga_norm;
  int64_t c;
  char note[128];
  /* per iteration: numerical rank of the COD of the cross block A(I,J) (threshold
     1e-12 * r, proj/src/pinv.cpp:54-60); < rank means the reference's core truncated (may be NULL) */
  int64_t* cod_rank;
} oracle_result;

const char* oracle_last_error(void);
/* Host threads used by the oracle's independent-column loops (results are bitwise independent of
   it); n < 1 restores all pool threads (ORACLE_THREADS or the hardware count). Returns the count. */
int oracle_set_threads(int n);

/* rng (proj/src/rng.cpp:30-67) */
void oracle_philox4x32(const uint32_t* ctr, const uint32_t* key, uint32_t* out);
double oracle_normal_at(uint64_t seed, uint32_t stream, int64_t i, int64_t j);
double oracle_uniform_at(uint64_t seed, uint32_t stream, int64_t i, int64_t j);
void oracle_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, uint32_t stream, double* out);
/* out(i, j) = scale * normal_at(seed, stream, i, j) + out(i, j) * keep  (col-major, ld = rows; threaded) */
void oracle_gaussian_fill(int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint32_t stream, double scale,
                          double* out);

/* sparse-sign stream (new): rows_out[i*zeta+t] = h_t(i), signs_out[i*zeta+t] = +-1 */
int oracle_sparse_sign_pattern(int64_t c, int64_t m, uint64_t seed, int32_t zeta, int32_t* rows_out,
                               int8_t* signs_out);

/* sketch (proj/src/sketch.cpp:10-24): Y = S*A, c x n column-major (ld = c). */
int64_t oracle_sketch_rows_for_block(int64_t b);
int oracle_sketch(const double* A, int64_t m, int64_t n, int64_t lda, int64_t b, uint64_t seed,
                  int32_t kind, int32_t zeta, double* Y, double* ga_norm, double* a_norm);

/* selection (proj/src/select.cpp:121-165). is_columns=1: select_columns(M, b), else select_rows. */
int oracle_select(const double* M, int64_t rows, int64_t cols, int64_t ldm, int64_t b, int32_t is_columns,
                  int32_t method, double pivot_floor, const int64_t* exclude, int64_t n_exclude,
                  int64_t* idx_out, int64_t* n_idx, int32_t* truncated, double* last_pivot,
                  double* best_out, double* second_out);

/* driver (proj/src/driver.cpp:28-190) */
int oracle_adjusted_threshold(double epsilon, double delta, double alpha, int64_t c, double* out);
int oracle_gratton_tail(int64_t c, double tau, double* out);
int oracle_iterative_cur(const double* A, int64_t m, int64_t n, int64_t lda, const oracle_config* cfg,
                         oracle_result* res);
int oracle_true_relative_error(const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I,
                               const int64_t* J, int64_t r, double* out);
/* core_out = A(I,J)^+ (r x r column-major), via the COD restatement (proj/src/pinv.cpp:40-65) */
int oracle_core_matrix(const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I,
                       const int64_t* J, int64_t r, double* core_out);

/* out = A(I,J)^+ * rhs (r x k, ld r) by the COD's minimum-norm solve (FactoredPinv::solve,
   proj/src/pinv.cpp:24-31) — what true_relative_error applies to R's panels (driver.cpp:183-185) */
int oracle_core_solve(const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I, const int64_t* J,
                      int64_t r, const double* rhs, int64_t k, int64_t ldrhs, double* out);

/* one-shot s-LUPP CUR baseline (proj/src/baselines.cpp:39-62): I, J (length *rank <= r) */
int oracle_slupp_cur(const double* A, int64_t m, int64_t n, int64_t lda, int64_t r, uint64_t seed, int64_t* I,
                     int64_t* J, int64_t* rank);

/* proj/tests/oracles.hpp:20-37 fixtures (std::mt19937_64 + libstdc++ distributions) */
void oracle_fixture_random_dense(int64_t rows, int64_t cols, uint32_t seed, double lo, double hi, double* out);
void oracle_fixture_random_gaussian(int64_t rows, int64_t cols, uint32_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif

// misc.h — small per-iteration kernels (misc.cu), the device-resident loop control and the
// per-iteration record.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace itercur_b200 {

// Loop state that lives on the device so the host can enqueue several iterations without
// waiting for each one (proj/src/driver.cpp:86-160 control flow, evaluated on the device).
struct IterCtl {
  int64_t r;          // current rank (sum of committed widths)
  int64_t k;          // committed iterations
  int64_t max_rank;
  int64_t max_iters;
  int32_t done;       // set once the run must stop; every later kernel returns immediately
  int32_t status;     // 0 Converged, 1 MaxRank, 2 ResidualExhausted (valid when done)
  int32_t block;      // requested column steps of the current iteration: min(b, max_rank - r)
  int32_t b;
  double ysq;         // ||Y||_F^2 of the current sketched residual
  double rho;         // ||Y||_F / ||GA||_F
  double threshold;
  double ga_norm;
};

// Device-side record of one iteration. Lives at the head of one allocation slot followed by
// six arrays of `b` entries (col_idx, row_idx as int64; col_best, col_second, row_best,
// row_second as double) so one D2H copy returns a whole batch of iterations.
struct IterState {
  int ncols;   // accepted column pivots (col LUPP)
  int nrows;   // accepted row pivots (row LUPP)
  int width;   // min(ncols, nrows)
  int valid;   // 1 if this slot's iteration ran (the run was not already done)
  double ysq;  // ||Y||_F^2 after the downdate
  double rho;  // ||Y||_F / ||GA||_F
  double pad2[4];
};
static_assert(sizeof(IterState) == 64, "IterState header is 64 bytes");

struct IterArrays {
  int64_t* col_idx;
  int64_t* row_idx;
  double* col_best;
  double* col_second;
  double* row_best;
  double* row_second;
};
// Everything an iteration commit touches (driver.cpp:102-159): run by commit_kernel, or by the
// last CTA of the fused U-block kernel (CommitArgs::counter, reset by that CTA).
struct CommitArgs {
  IterCtl* ctl = nullptr;
  IterState* slot = nullptr;
  const int64_t* row_idx = nullptr;
  const int64_t* col_idx = nullptr;
  int64_t* I_all = nullptr;
  int64_t* J_all = nullptr;
  uint8_t* row_mask = nullptr;
  uint8_t* col_mask = nullptr;
  int* counter = nullptr;  // fused form only
};
#ifdef __CUDACC__
}  // namespace itercur_b200
#include "common.cuh"
namespace itercur_b200 {
// One CTA of THREADS threads: ||Y||^2 from the per-CTA partials in a fixed order, the stop
// tests, the index append and the masks. `red` holds THREADS / 32 doubles.
template <int THREADS>
__device__ inline void commit_body(const CommitArgs& c, const double* __restrict__ y_partials, int64_t y_parts,
                                   double* red) {
  __shared__ int s_stop;
  IterCtl* ctl = c.ctl;
  IterState* slot = c.slot;
  {  // ||Y||^2 of the downdated residual: fixed-order sum of the GEMM's per-CTA partials
    double sq = 0.0;
    for (int64_t i = threadIdx.x; i < y_parts; i += THREADS) sq += y_partials[i];
    const double tot = block_sum<THREADS>(sq, red);
    if (threadIdx.x == 0) ctl->ysq = tot;
  }
  const int width = min(slot->ncols, slot->nrows);
  const int64_t r = ctl->r;
  if (threadIdx.x == 0) s_stop = (slot->ncols == 0 || slot->nrows == 0) ? 1 : 0;
  __syncthreads();
  if (s_stop) {  // empty column or row selection -> ResidualExhausted, factors unchanged
    if (threadIdx.x == 0) {
      ctl->done = 1;
      ctl->status = 2;
    }
    return;
  }
  for (int q = threadIdx.x; q < width; q += THREADS) {
    c.I_all[r + q] = c.row_idx[q];
    c.J_all[r + q] = c.col_idx[q];
    c.row_mask[c.row_idx[q]] = 1;
    c.col_mask[c.col_idx[q]] = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double rho = ctl->ga_norm > 0.0 ? sqrt(ctl->ysq) / ctl->ga_norm : 0.0;
    slot->width = width;
    slot->ysq = ctl->ysq;
    slot->rho = rho;
    ctl->rho = rho;
    ctl->r = r + width;
    ctl->k += 1;
    if (rho <= ctl->threshold) {
      ctl->done = 1;
      ctl->status = 0;  // Converged
    }
  }
}
#endif

inline size_t iter_state_bytes(int b) { return sizeof(IterState) + 6 * sizeof(double) * static_cast<size_t>(b); }
inline IterArrays iter_arrays(void* base, int b) {
  char* p = static_cast<char*>(base) + sizeof(IterState);
  IterArrays a;
  a.col_idx = reinterpret_cast<int64_t*>(p);
  a.row_idx = a.col_idx + b;
  a.col_best = reinterpret_cast<double*>(a.row_idx + b);
  a.col_second = a.col_best + b;
  a.row_best = a.col_second + b;
  a.row_second = a.row_best + b;
  return a;
}

cudaError_t launch_transpose_rows(const double* Y, int64_t cp, int64_t n, int rows, double* Wc, int64_t ldwc,
                                  cudaStream_t st);
// At(j, i) = A(i, j) (At column-major n x m, ld ldt): the engine's row-major copy of A
cudaError_t launch_transpose(const double* A, int64_t m, int64_t n, int64_t lda, double* At, int64_t ldt,
                             cudaStream_t st);
// out(k, q) = src[k * row_stride + idx[q] * col_stride] for k < K, q < min(*d_w, w_max), zero for
// q >= w. With ctl: skipped when ctl->done, and K = ctl->r when k_from_r.
cudaError_t launch_gather_pair(const double* src0, int64_t rs0, int64_t cs0, int64_t K0, const int64_t* idx0,
                               double* out0, int64_t ldo0, bool k_from_r0, const double* src1, int64_t rs1,
                               int64_t cs1, int64_t K1, const int64_t* idx1, double* out1, int64_t ldo1,
                               bool k_from_r1, const int* d_w, int w_max, cudaStream_t st, const IterCtl* ctl);
cudaError_t launch_gather(const double* src, int64_t row_stride, int64_t col_stride, int64_t K, const int64_t* d_idx,
                          const int* d_w, int w_max, double* out, int64_t ldo, cudaStream_t st,
                          const IterCtl* ctl = nullptr, bool k_from_r = false, bool transposed = false);
// out(k, q) = src[idx[k] + q * ld] for k < K, q < w (row-indexed gather)
cudaError_t launch_gather2(const double* src, int64_t ld, const int64_t* d_idx, int64_t K, int w, double* out,
                           int64_t ldo, cudaStream_t st);
// G(i, j) = normal_at(seed, stream_tag, i, j), rows x cols column-major (rng.cpp:61-67)
cudaError_t launch_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, uint32_t stream_tag, double* out,
                                   cudaStream_t st);
// LU of D = Lk(rows, 0:w) into lu (ld ldd): without pivoting (rows already in LUPP order), or,
// with `perm`, partial pivoting P D = Lhat Uhat (perm[q] = row of D at position q).
// With ctl: Lk += ctl->r * ldl, lu += ctl->r * ldd, perm += ctl->r, skipped when done.
cudaError_t launch_cross_lu(const double* Lk, int64_t ldl, const int64_t* d_rows, const int* d_w, int w_max,
                            double* lu, int64_t ldd, cudaStream_t st, const IterCtl* ctl = nullptr,
                            int* perm = nullptr);
// out(j, :) = X(j, :) * D^{-T} (each row solves D x = u) via the LU factors (in place allowed);
// with `perm` the factors are of P D and u is loaded permuted. Any width (w > 168: factors read
// from global memory). With ctl: lu += ctl->r * ldd, perm += ctl->r, out += ctl->r * out_off_per_r,
// skipped when done.
cudaError_t launch_rows_lu_solve(const double* X, int64_t ldx, int64_t M, const double* lu, int64_t ldd,
                                 const int* d_w, int w_max, double* out, int64_t ldo, cudaStream_t st,
                                 const IterCtl* ctl = nullptr, int64_t out_off_per_r = 0,
                                 const int* perm = nullptr);
// Column-sharded engine: this shard's columns of the selected block J_k into the packed block
// [A(:, J_k) | R~(0:r, J_k) | Y(:, J_k)] (misc.cu pack_owned_kernel); zero_rest for a sum-allreduce.
cudaError_t launch_pack_owned(const IterCtl* ctl, const int* d_ncols, const int64_t* col_idx, int B, int64_t goff,
                              int64_t cnt, const double* A, int64_t lda, int64_t m, const double* Rt, int64_t ldR,
                              int64_t r_cap, const double* Y, int64_t cp, double* PackA, int64_t ldpa, double* PackR,
                              int64_t ldpr, double* PackY, bool zero_rest, cudaStream_t st);
cudaError_t launch_sum_partials(const double* partials, int64_t count, double* d_out, cudaStream_t st,
                                const IterCtl* ctl = nullptr);
cudaError_t launch_sumsq(const double* x, int64_t rows, int64_t cols, int64_t ld, double* partials, int max_parts,
                         double* d_out, cudaStream_t st);
cudaError_t launch_count_nonfinite(const double* x, int64_t rows, int64_t cols, int64_t ld,
                                   unsigned long long* d_count, cudaStream_t st);
// Start of an iteration (driver.cpp:87-95): budget checks, block = min(b, max_rank - r).
cudaError_t launch_iter_begin(IterCtl* ctl, IterState* slot, cudaStream_t st);
// width = min(ncols, nrows) (driver.cpp:123), published before the core/downdate stages.
cudaError_t launch_width(IterState* slot, const IterCtl* ctl, cudaStream_t st);
// End of an iteration (driver.cpp:102-159): empty selections -> ResidualExhausted; append the
// first `width` pivots to I, J, ban them, r += width, k++, rho = ||Y||/||GA||, rho <= thr ->
// Converged.
// The ||Y||^2 partials of the downdate (y_parts of them) are summed here in a fixed order.
cudaError_t launch_commit(IterCtl* ctl, IterState* slot, const IterArrays& arr, int64_t* I_all, int64_t* J_all,
                          uint8_t* row_mask, uint8_t* col_mask, const double* y_partials, int64_t y_parts,
                          cudaStream_t st);

cudaError_t launch_csr_to_dense(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                                double* out, int64_t ld, cudaStream_t st);

}  // namespace itercur_b200

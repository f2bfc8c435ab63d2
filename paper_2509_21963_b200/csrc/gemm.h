// gemm.h — parameters of the tall-skinny DMMA GEMM (gemm.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"
#include "misc.h"

namespace itercur_b200 {

enum GemmBase {
  kBaseNone = 0,
  kBaseGatherCols = 1,
  kBaseGatherRowsT = 2,
  kBaseContigCols = 3,
  kBaseInPlaceRowMajor = 4,
  kBaseIdentityCols = 5  // base(i, q) = (i == col0 + q)
};
enum GemmOut { kOutNone = 0, kOutColMajor = 1, kOutRowMajor = 2 };

// C(M x N) = base(M x N) + alpha * Aop(M x K) * B(K x N)
//   Aop(i, k) = A[i + k * lda]        (lda even, A 16-byte aligned)
//   B(k, q)   = B[k * bsk + q * bsn]
//   base: none | src(i, idx[q]) | src(idx[q], i) | src(i, col0 + q) | C0(i, q) row-major
//   out:  none (norm only) | C0/C1 column-major | C0 row-major (+ Wc(i, q) = C for q < wc_rows)
struct TsGemmParams {
  int64_t M = 0, K = 0;
  const int* d_k = nullptr;  // optional dynamic cap on K (device int)
  int N = 0;               // columns (host bound); grid.y covers N in chunks of 8*NT
  const int* d_n = nullptr;  // optional dynamic cap on N (device int)
  const double* A = nullptr;
  int64_t lda = 0;
  const double* B = nullptr;
  int64_t bsk = 0, bsn = 0;
  const int64_t* b_idx = nullptr;  // optional: B(k, q) = B[k * bsk + b_idx[q] * bsn]
  int base_mode = kBaseNone;
  const double* src = nullptr;
  int64_t lds = 0;
  const int64_t* idx = nullptr;
  int64_t col0 = 0;
  double alpha = -1.0;
  int out_mode = kOutColMajor;
  double* C0 = nullptr;
  int64_t ldc0 = 0;
  double* C1 = nullptr;
  int64_t ldc1 = 0;
  double* Wc = nullptr;
  int64_t ldwc = 0;
  int wc_rows = 0;
  double* norm_part = nullptr;  // [grid.y * grid.x] per-CTA sum of squares of C
  // device-resident loop control: skip when ctl->done; K = min(K, ctl->r) when k_from_r;
  // A += ctl->r * a_off_per_r and C0 += ctl->r * c0_off_per_r (elements)
  const IterCtl* ctl = nullptr;
  CommitArgs commit;        // U block: when commit.ctl is set, the last CTA also commits the iteration
  int64_t k_plan = 0;        // host-side hint: the K the split count is planned for (0: K)
  int64_t dbg_k = 0;         // ... recorded at iteration ctl->k == dbg_k
  int early_base = -1;       // base values loaded before the main loop (-1: by width, see gemm.cu)
  long long* dbg = nullptr;  // optional trace (U block): [0..15] clock64 phases of CTA (0,0,0); [32+2c] globaltimer entry/exit of CTA c
  int k_from_r = 0;
  int64_t a_off_per_r = 0;
  int64_t c0_off_per_r = 0;
  // fused U-block epilogue (run_ts_gemm_ublock; N = w <= 32): C = U_k^T rows, then per row j
  //   x_j = D_k^{-1} u_j   (LU solves with the factors at lu + r*ldd, w x w, pitch ldd)
  //   R~(r+q, j) = x_j[q]  (rt[(r+q)*ldr + j])
  //   Y^T(j, :) -= x_j^T Y(:, J_k)^T   (y row-major n x ycp, yg[h + q*ycp] = Y(h, J_k[q]))
  //   Wc(j, h) = Y^T(j, h) for h < wc_rows, norm_part = per-CTA sum of squares of the new Y^T
  const double* lu = nullptr;
  int64_t ldd = 0;
  double* rt = nullptr;
  int64_t ldr = 0;
  const double* yg = nullptr;
  int ycp = 0;
  double* y = nullptr;
};

cudaError_t run_ts_gemm(const TsGemmParams& p, cudaStream_t st);
int64_t ts_gemm_grid_size(int64_t M, int N);
// grid.z (K splits) the launch of these parameters would use (no launch)
int ts_gemm_planned_splits(const TsGemmParams& p, bool ublock);
// the fused U-block GEMM: returns cudaErrorNotSupported when the shape / layout does not
// qualify (the caller then runs GEMM + rows_lu_solve + downdate GEMM separately)
bool ts_gemm_ublock_supported(const TsGemmParams& p);
cudaError_t run_ts_gemm_ublock(const TsGemmParams& p, cudaStream_t st);
int64_t ts_gemm_ublock_parts(int64_t M);

}  // namespace itercur_b200

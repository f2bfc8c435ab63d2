// misc.cu — small per-iteration kernels: gathers of the selected rows/columns
// (proj/src/matrix.cpp:134-227 gather_cols / gather_rows / gather_block), the w x w
// cross-block inverse D_k^{-1} (the reference's per-iteration COD of the r x r cross
// block, proj/src/pinv.cpp:45-65, becomes an O(w^3) block step), deterministic norm
// reductions and the iteration commit (index append, masks, rho = ||Y||/||GA||,
// proj/src/sketch.cpp:40 and proj/src/driver.cpp:123-159).
#include <algorithm>

#include "common.cuh"
#include "misc.h"

namespace itercur_b200 {

namespace {
thread_local bool g_pdl = false;
}
bool pdl_enabled() { return g_pdl; }
PdlScope::PdlScope(bool on) : prev(g_pdl) { g_pdl = on; }
PdlScope::~PdlScope() { g_pdl = prev; }

// Wc(j, h) = Y(h, j) for h < rows  (Wc column-major n x rows)
__global__ void transpose_rows_kernel(const double* __restrict__ Y, int64_t cp, int64_t n, int rows,
                                      double* __restrict__ Wc, int64_t ldwc) {
  const int64_t total = n * rows;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = e / n, j = e - h * n;
    Wc[j + h * ldwc] = Y[h + j * cp];
  }
}

// At(j, i) = A(i, j): 32 x 32 tiles through shared memory (both sides coalesced), one pass of
// 16 bytes per element over HBM. The engine keeps this row-major copy of A so the row gathers
// A(I_k, :) of the U block read contiguous rows instead of one DRAM burst per element.
__global__ void __launch_bounds__(256) transpose_tiled_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                                                              int64_t lda, double* __restrict__ At, int64_t ldt) {
  __shared__ double tile[32][33];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, j0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int64_t i = i0 + tx, j = j0 + ty + r;
    if (i < m && j < n) tile[ty + r][tx] = A[i + j * lda];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int64_t j = j0 + tx, i = i0 + ty + r;
    if (i < m && j < n) At[j + i * ldt] = tile[tx][ty + r];
  }
}

cudaError_t launch_transpose(const double* A, int64_t m, int64_t n, int64_t lda, double* At, int64_t ldt,
                             cudaStream_t st) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  if (ceil_div(n, 32) > 65535) return cudaErrorInvalidValue;
  transpose_tiled_kernel<<<dim3(static_cast<unsigned>(ceil_div(m, 32)), static_cast<unsigned>(ceil_div(n, 32))), 256, 0,
                           st>>>(A, m, n, lda, At, ldt);
  return cudaGetLastError();
}

// out(k, q) = src[k * row_stride + idx[q] * col_stride] for k < K, q < w (dynamic), zero for q >= w
__global__ void gather_kernel(const double* __restrict__ src, int64_t row_stride, int64_t col_stride, int64_t Kmax,
                              const int64_t* __restrict__ idx, const int* __restrict__ d_w, int w_max,
                              double* __restrict__ out, int64_t ldo, const IterCtl* __restrict__ ctl, int k_from_r,
                              int transposed) {
  griddep_wait();
  griddep_launch_dependents();
  if (ctl && ctl->done) return;
  const int64_t K = (ctl && k_from_r) ? min(Kmax, ctl->r) : Kmax;
  const int w = d_w ? min(*d_w, w_max) : w_max;
  const int64_t total = K * w_max;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / K, k = e - q * K;
    const double v = q < w ? src[k * row_stride + idx[q] * col_stride] : 0.0;
    if (transposed)
      out[q + k * ldo] = v;  // index-list dimension contiguous (a k-contiguous GEMM B operand)
    else
      out[k + q * ldo] = v;
  }
}

cudaError_t launch_transpose_rows(const double* Y, int64_t cp, int64_t n, int rows, double* Wc, int64_t ldwc,
                                  cudaStream_t st) {
  const int64_t total = n * rows;
  if (total <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 148 * 8));
  transpose_rows_kernel<<<blocks, 256, 0, st>>>(Y, cp, n, rows, Wc, ldwc);
  return cudaGetLastError();
}

cudaError_t launch_gather(const double* src, int64_t row_stride, int64_t col_stride, int64_t K, const int64_t* d_idx,
                          const int* d_w, int w_max, double* out, int64_t ldo, cudaStream_t st, const IterCtl* ctl,
                          bool k_from_r, bool transposed) {
  const int64_t total = K * w_max;
  if (total <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 148 * 8));
  return launch_ex(gather_kernel, dim3(blocks), dim3(256), 0, st, dim3(0, 0, 0), src, row_stride, col_stride, K, d_idx,
                   d_w, w_max, out, ldo, ctl, k_from_r ? 1 : 0, transposed ? 1 : 0);
}

// Two gathers of the same (dynamic) width in one launch: the U block's operands L(I_k, :)^T and
// Y(:, J_k) (one launch per iteration fewer inside the batch graphs)
struct GatherDesc {
  const double* src;
  int64_t row_stride, col_stride, Kmax;
  const int64_t* idx;
  double* out;
  int64_t ldo;
  int k_from_r;
};
__global__ void gather_pair_kernel(GatherDesc g0, GatherDesc g1, const int* __restrict__ d_w, int w_max,
                                   const IterCtl* __restrict__ ctl) {
  griddep_wait();
  griddep_launch_dependents();
  if (ctl && ctl->done) return;
  const int w = d_w ? min(*d_w, w_max) : w_max;
  const int64_t K0 = (ctl && g0.k_from_r) ? min(g0.Kmax, ctl->r) : g0.Kmax;
  const int64_t K1 = (ctl && g1.k_from_r) ? min(g1.Kmax, ctl->r) : g1.Kmax;
  const int64_t t0 = K0 * w_max, total = t0 + K1 * w_max;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const bool second = e >= t0;
    const GatherDesc& g = second ? g1 : g0;
    const int64_t K = second ? K1 : K0, f = second ? e - t0 : e;
    const int64_t q = f / K, k = f - q * K;
    g.out[k + q * g.ldo] = q < w ? g.src[k * g.row_stride + g.idx[q] * g.col_stride] : 0.0;
  }
}
cudaError_t launch_gather_pair(const double* src0, int64_t rs0, int64_t cs0, int64_t K0, const int64_t* idx0,
                               double* out0, int64_t ldo0, bool k_from_r0, const double* src1, int64_t rs1,
                               int64_t cs1, int64_t K1, const int64_t* idx1, double* out1, int64_t ldo1,
                               bool k_from_r1, const int* d_w, int w_max, cudaStream_t st, const IterCtl* ctl) {
  const int64_t total = (K0 + K1) * w_max;
  if (total <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 148 * 8));
  const GatherDesc g0{src0, rs0, cs0, K0, idx0, out0, ldo0, k_from_r0 ? 1 : 0};
  const GatherDesc g1{src1, rs1, cs1, K1, idx1, out1, ldo1, k_from_r1 ? 1 : 0};
  return launch_ex(gather_pair_kernel, dim3(blocks), dim3(256), 0, st, dim3(0, 0, 0), g0, g1, d_w, w_max, ctl);
}

__global__ void gather2_kernel(const double* __restrict__ src, int64_t ld, const int64_t* __restrict__ idx, int64_t K,
                               int w, double* __restrict__ out, int64_t ldo) {
  const int64_t total = K * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / K, k = e - q * K;
    out[k + q * ldo] = src[idx[k] + q * ld];
  }
}
cudaError_t launch_gather2(const double* src, int64_t ld, const int64_t* d_idx, int64_t K, int w, double* out,
                           int64_t ldo, cudaStream_t st) {
  const int64_t total = K * w;
  if (total <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 148 * 8));
  gather2_kernel<<<blocks, 256, 0, st>>>(src, ld, d_idx, K, w, out, ldo);
  return cudaGetLastError();
}

__global__ void gaussian_matrix_kernel(int64_t rows, int64_t cols, uint64_t seed, uint32_t tag, double* __restrict__ out) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    out[e] = normal_at_dev(seed, tag, i, j);
  }
}
cudaError_t launch_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, uint32_t stream_tag, double* out,
                                   cudaStream_t st) {
  const int64_t total = rows * cols;
  if (total <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 148 * 16));
  gaussian_matrix_kernel<<<blocks, 256, 0, st>>>(rows, cols, seed, stream_tag, out);
  return cudaGetLastError();
}

// D(p, q) = L_k(I_k[p], q) for p, q < w. Doolittle LU without pivoting — the rows are
// already in LUPP pivot order, so these are exactly the row-LUPP's eliminations. The
// factors (unit-lower multipliers below the diagonal, U on and above) stay in `lu`; the
// block is never inverted explicitly (an explicit inverse loses accuracy in proportion to
// cond(D_k), which reaches 1e9+ once pivots hit the noise floor).
//
// With `perm` (row selections that are not LUPP-ordered, e.g. QRCP rows): partial pivoting,
// P D = Lhat Uhat with perm[q] = the row of D placed at position q (largest |entry| in the
// column, lowest index on ties) — the reference's COD (pinv.cpp:54-58) accepts any
// nonsingular cross block, and QRCP's order can put an exact zero on D's diagonal.
__global__ void cross_lu_kernel(const double* __restrict__ Lk, int64_t ldl, const int64_t* __restrict__ rows,
                                const int* __restrict__ d_w, int w_max, double* __restrict__ lu, int64_t ldd,
                                const IterCtl* __restrict__ ctl, int* __restrict__ perm) {
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  griddep_wait();
  griddep_launch_dependents();
  if (ctl) {
    if (ctl->done) return;
    Lk += ctl->r * ldl;
    lu += ctl->r * ldd;
    if (perm) perm += ctl->r;
  }
  const int w = min(*d_w, w_max);
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
    const int p = e % w, q = e / w;
    lu[p + q * ldd] = Lk[rows[p] + q * ldl];
  }
  if (perm)
    for (int q = threadIdx.x; q < w; q += blockDim.x) perm[q] = q;
  __syncthreads();
  for (int s = 0; s < w; ++s) {
    if (perm) {  // argmax |lu(p, s)|, p >= s (lowest index on ties), then swap rows s and p
      double bv = -1.0;
      int bi = w;
      for (int p = s + threadIdx.x; p < w; p += blockDim.x) {
        const double v = fabs(lu[p + s * ldd]);
        if (v > bv) { bv = v; bi = p; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if ((threadIdx.x & 31) == 0) { red_v[threadIdx.x >> 5] = bv; red_i[threadIdx.x >> 5] = bi; }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int q = 1; q < static_cast<int>(blockDim.x >> 5); ++q)
          if (red_v[q] > red_v[0] || (red_v[q] == red_v[0] && red_i[q] < red_i[0])) { red_v[0] = red_v[q]; red_i[0] = red_i[q]; }
      }
      __syncthreads();
      const int p = red_i[0];
      if (p != s && p < w) {
        for (int t = threadIdx.x; t < w; t += blockDim.x) {
          const double x = lu[s + t * ldd];
          lu[s + t * ldd] = lu[p + t * ldd];
          lu[p + t * ldd] = x;
        }
        if (threadIdx.x == 0) {
          const int x = perm[s];
          perm[s] = perm[p];
          perm[p] = x;
        }
      }
      __syncthreads();
    }
    const double piv = lu[s + s * ldd];
    const int rem = w - s - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      const int p = s + 1 + e % rem;
      const int tq = s + 1 + e / rem;
      const double f = __ddiv_rn(lu[p + s * ldd], piv);
      lu[p + tq * ldd] = __dsub_rn(lu[p + tq * ldd], __dmul_rn(f, lu[s + tq * ldd]));
    }
    __syncthreads();
    for (int p = s + 1 + threadIdx.x; p < w; p += blockDim.x) lu[p + s * ldd] = __ddiv_rn(lu[p + s * ldd], piv);
    __syncthreads();
  }
}

// One-warp variant for w <= 32: lane p holds row p of D in registers; the pivot row is
// broadcast with shuffles (same operations and roundings as cross_lu_kernel).
__global__ void cross_lu_warp_kernel(const double* __restrict__ Lk, int64_t ldl, const int64_t* __restrict__ rows,
                                     const int* __restrict__ d_w, double* __restrict__ lu, int64_t ldd,
                                     const IterCtl* __restrict__ ctl) {
  griddep_wait();
  griddep_launch_dependents();
  if (ctl) {
    if (ctl->done) return;
    Lk += ctl->r * ldl;
    lu += ctl->r * ldd;
  }
  const int w = min(*d_w, 32);
  const int lane = threadIdx.x;
  double d[32];
  const int64_t row = lane < w ? rows[lane] : 0;
#pragma unroll
  for (int t = 0; t < 32; ++t) d[t] = (lane < w && t < w) ? Lk[row + t * ldl] : 0.0;
#pragma unroll
  for (int s = 0; s < 32; ++s) {
    if (s < w) {
      const double piv = __shfl_sync(0xffffffffu, d[s], s);
      const bool below = lane > s && lane < w;
      const double f = below ? __ddiv_rn(d[s], piv) : 0.0;
#pragma unroll
      for (int t = s + 1; t < 32; ++t) {
        const double pt = __shfl_sync(0xffffffffu, d[t], s);
        if (below && t < w) d[t] = __dsub_rn(d[t], __dmul_rn(f, pt));
      }
      if (below) d[s] = f;
    }
  }
  if (lane < w) {
#pragma unroll
    for (int t = 0; t < 32; ++t)
      if (t < w) lu[lane + t * ldd] = d[t];
  }
}

cudaError_t launch_cross_lu(const double* Lk, int64_t ldl, const int64_t* d_rows, const int* d_w, int w_max,
                            double* lu, int64_t ldd, cudaStream_t st, const IterCtl* ctl, int* perm) {
  if (w_max <= 32 && !perm)
    return launch_ex(cross_lu_warp_kernel, dim3(1), dim3(32), 0, st, dim3(0, 0, 0), Lk, ldl, d_rows, d_w, lu, ldd, ctl);
  return launch_ex(cross_lu_kernel, dim3(1), dim3(256), 0, st, dim3(0, 0, 0), Lk, ldl, d_rows, d_w, w_max, lu, ldd, ctl,
                   perm);
}

// Row-wise solves D x = u with D = Lhat * Uhat (cross_lu_kernel layout) for every row u of
// X (M x w, column-major), i.e. out = X * D^{-T}: forward substitution with the unit-lower
// Lhat, then back substitution with Uhat. One thread per row; the factors sit in shared
// memory. Backward stable, unlike multiplying by an explicit D^{-1}.
template <int WMAX>
__global__ void rows_lu_solve_kernel(const double* __restrict__ X, int64_t ldx, int64_t M,
                                     const double* __restrict__ lu, int64_t ldd, const int* __restrict__ d_w,
                                     int w_max, double* __restrict__ out, int64_t ldo,
                                     const IterCtl* __restrict__ ctl, int64_t out_off_per_r,
                                     const int* __restrict__ perm) {
  extern __shared__ double slu[];
  __shared__ int sperm[WMAX];
  griddep_wait();
  griddep_launch_dependents();
  if (ctl) {
    if (ctl->done) return;
    lu += ctl->r * ldd;
    out += ctl->r * out_off_per_r;
    if (perm) perm += ctl->r;
  }
  const int w = d_w ? min(*d_w, w_max) : w_max;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) slu[e] = lu[(e % w) + (e / w) * ldd];
  for (int q = threadIdx.x; q < WMAX; q += blockDim.x) sperm[q] = (perm && q < w) ? perm[q] : q;
  __syncthreads();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
    double x[WMAX];  // fully unrolled: stays in registers
#pragma unroll
    for (int q = 0; q < WMAX; ++q) x[q] = q < w ? X[j + sperm[q] * ldx] : 0.0;  // P u (perm: pivoted LU)
#pragma unroll
    for (int q = 1; q < WMAX; ++q) {  // Lhat y = u
      if (q < w) {
        double v = x[q];
#pragma unroll
        for (int p = 0; p < q; ++p) v = fma(-slu[q + p * w], x[p], v);
        x[q] = v;
      }
    }
#pragma unroll
    for (int q = WMAX - 1; q >= 0; --q) {  // Uhat x = y
      if (q < w) {
        double v = x[q];
#pragma unroll
        for (int p = q + 1; p < WMAX; ++p)
          if (p < w) v = fma(-slu[q + p * w], x[p], v);
        x[q] = v / slu[q + q * w];
      }
    }
#pragma unroll
    for (int q = 0; q < WMAX; ++q)
      if (q < w) out[j + q * ldo] = x[q];
  }
}

// Column-oriented form of the same solves for 16 < w <= WMAX, a row shared by a lane pair (lane
// bit 0 = which half of the row): the outer loop over pivots p is a runtime loop and only the
// update over the thread's WMAX/2 entries is unrolled, so every register index is static (the
// row-oriented kernel above keeps its fully unrolled triangle in local memory beyond 16 columns:
// 255 registers + a 560-byte stack frame at WMAX = 64). x[p] is read with a static select and
// handed to the partner with one shuffle. The forward substitution updates each x[q] in
// ascending p, exactly as the row form; the back substitution updates x[q] in descending p (a
// different, equally backward-stable rounding order).
template <int WMAX>
__global__ void __launch_bounds__(128) rows_lu_solve_col_kernel(const double* __restrict__ X, int64_t ldx, int64_t M,
                                                                const double* __restrict__ lu, int64_t ldd,
                                                                const int* __restrict__ d_w, int w_max,
                                                                double* __restrict__ out, int64_t ldo,
                                                                const IterCtl* __restrict__ ctl, int64_t out_off_per_r,
                                                                const int* __restrict__ perm) {
  constexpr int H = WMAX / 2;
  extern __shared__ double slu[];
  __shared__ int sperm[WMAX];
  griddep_wait();
  griddep_launch_dependents();
  if (ctl) {
    if (ctl->done) return;
    lu += ctl->r * ldd;
    out += ctl->r * out_off_per_r;
    if (perm) perm += ctl->r;
  }
  const int w = d_w ? min(*d_w, w_max) : w_max;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) slu[e] = lu[(e % w) + (e / w) * ldd];
  for (int q = threadIdx.x; q < WMAX; q += blockDim.x) sperm[q] = (perm && q < w) ? perm[q] : q;
  __syncthreads();
  const int half = threadIdx.x & 1;
  const int q0 = half * H;  // this thread's entries: q0 .. q0 + H - 1
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 1);
  const int64_t rows_pad = ceil_div(M, stride) * stride;  // pairs stay converged: both lanes loop alike
  for (int64_t j = blockIdx.x * (int64_t)(blockDim.x >> 1) + (threadIdx.x >> 1); j < rows_pad; j += stride) {
    const bool live = j < M;
    double x[H];
#pragma unroll
    for (int q = 0; q < H; ++q) x[q] = (live && q0 + q < w) ? X[j + sperm[q0 + q] * ldx] : 0.0;  // P u
    for (int p = 0; p + 1 < w; ++p) {  // Lhat y = u (unit lower)
      double mine = 0.0;
#pragma unroll
      for (int q = 0; q < H; ++q) mine = q0 + q == p ? x[q] : mine;
      const double other = __shfl_xor_sync(0xffffffffu, mine, 1);
      const double xp = (p >= q0 && p < q0 + H) ? mine : other;
      const double* col = slu + p * w;
#pragma unroll
      for (int q = 0; q < H; ++q)
        if (q0 + q > p && q0 + q < w) x[q] = fma(-col[q0 + q], xp, x[q]);
    }
    for (int p = w - 1; p >= 0; --p) {  // Uhat x = y
      double mine = 0.0;
#pragma unroll
      for (int q = 0; q < H; ++q) mine = q0 + q == p ? x[q] : mine;
      const double other = __shfl_xor_sync(0xffffffffu, mine, 1);
      const double xp = ((p >= q0 && p < q0 + H) ? mine : other) / slu[p + p * w];
#pragma unroll
      for (int q = 0; q < H; ++q) x[q] = q0 + q == p ? xp : x[q];
      const double* col = slu + p * w;
#pragma unroll
      for (int q = 0; q < H; ++q)
        if (q0 + q < p) x[q] = fma(-col[q0 + q], xp, x[q]);
    }
    if (live) {
#pragma unroll
      for (int q = 0; q < H; ++q)
        if (q0 + q < w) out[j + (q0 + q) * ldo] = x[q];
    }
  }
}

// The row-oriented solves with each thread's row in SHARED memory (xs[q][thread]: consecutive
// threads, consecutive banks) and runtime loops: the register-array form above ends up in local
// memory beyond 16 columns and is latency-bound there (250 us at 100000 rows x 50); here the only
// dependency chain is the FMA accumulation of v (the loads of x[p] and L(q, p) are independent of
// it). Same operations in the same order as rows_lu_solve_kernel: bitwise its results.
template <int WMAX>
__global__ void __launch_bounds__(128) rows_lu_solve_smem_kernel(const double* __restrict__ X, int64_t ldx, int64_t M,
                                                                 const double* __restrict__ lu, int64_t ldd,
                                                                 const int* __restrict__ d_w, int w_max,
                                                                 double* __restrict__ out, int64_t ldo,
                                                                 const IterCtl* __restrict__ ctl, int64_t out_off_per_r,
                                                                 const int* __restrict__ perm) {
  extern __shared__ double sm[];
  double* slu = sm;                 // w x w factors (ld w)
  double* xs = sm + WMAX * WMAX;    // xs[q * 128 + tid]
  __shared__ int sperm[WMAX];
  griddep_wait();
  griddep_launch_dependents();
  if (ctl) {
    if (ctl->done) return;
    lu += ctl->r * ldd;
    out += ctl->r * out_off_per_r;
    if (perm) perm += ctl->r;
  }
  const int w = d_w ? min(*d_w, w_max) : w_max;
  for (int e = threadIdx.x; e < w * w; e += blockDim.x) slu[e] = lu[(e % w) + (e / w) * ldd];
  for (int q = threadIdx.x; q < WMAX; q += blockDim.x) sperm[q] = (perm && q < w) ? perm[q] : q;
  __syncthreads();
  double* x = xs + threadIdx.x;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
    for (int q = 0; q < w; ++q) x[q * 128] = X[j + sperm[q] * ldx];  // P u
    for (int q = 1; q < w; ++q) {  // Lhat y = u
      double v = x[q * 128];
      const double* lq = slu + q;
#pragma unroll 4
      for (int p = 0; p < q; ++p) v = fma(-lq[p * w], x[p * 128], v);
      x[q * 128] = v;
    }
    for (int q = w - 1; q >= 0; --q) {  // Uhat x = y
      double v = x[q * 128];
      const double* lq = slu + q;
#pragma unroll 4
      for (int p = q + 1; p < w; ++p) v = fma(-lq[p * w], x[p * 128], v);
      x[q * 128] = v / slu[q + q * w];
    }
    for (int q = 0; q < w; ++q) out[j + q * ldo] = x[q * 128];
  }
}

// Tensor-core form (default for 16 < w <= 64): R~_k rows = the rows of U_k^T solved against
// D_k = Lhat Uhat, as a blocked triangular solve on DMMA. A warp owns 16 rows as the C fragments
// of ceil(w/8) column chunks; chunk P is first updated by every finished chunk Q with one
// m16n8k8 per (P, Q) pair — the finished chunk's C fragment is the A operand as it stands (the
// k permutation logical t <-> column 2t, t+4 <-> 2t+1 of the GEMMs), B = -L(P, Q)^T staged in
// shared memory — then solved within its 8 x 8 diagonal block by substitution on the fragment
// (the row's 8 entries live in a quad: x_p broadcast with shuffles). Division by U's diagonal
// through its correctly rounded reciprocal (Markstein; IEEE division for the warp outside the
// safe exponent window), i.e. the IEEE quotient. Backward-stable like the row substitutions it
// replaces (no explicit inverse: D_k's condition number reaches 1e9+ near the noise floor).
template <int NT>
__global__ void __launch_bounds__(128) rows_lu_solve_mma_kernel(const double* __restrict__ X, int64_t ldx, int64_t M,
                                                                const double* __restrict__ lu, int64_t ldd,
                                                                const int* __restrict__ d_w, int w_max,
                                                                double* __restrict__ out, int64_t ldo,
                                                                const IterCtl* __restrict__ ctl, int64_t out_off_per_r,
                                                                const int* __restrict__ perm) {
  constexpr int W = NT * 8, WP = W + 4;  // negated factors, row pitch WP (16-byte fragment loads)
  __shared__ __align__(16) double sneg[W * WP];  // sneg[q * WP + p] = -LU(q, p), identity-padded
  __shared__ double srcp[W];                     // RN(1 / U(p, p))
  __shared__ int sperm[W];
  griddep_wait();
  griddep_launch_dependents();
  if (ctl) {
    if (ctl->done) return;
    lu += ctl->r * ldd;
    out += ctl->r * out_off_per_r;
    if (perm) perm += ctl->r;
  }
  const int w = d_w ? min(*d_w, w_max) : w_max;
  for (int e = threadIdx.x; e < W * W; e += 128) {
    const int q = e % W, p = e / W;
    const double v = (q < w && p < w) ? lu[q + p * ldd] : (q == p ? 1.0 : 0.0);
    sneg[q * WP + p] = -v;
  }
  for (int p = threadIdx.x; p < W; p += 128) {
    srcp[p] = p < w ? __drcp_rn(lu[p + p * ldd]) : 1.0;
    sperm[p] = (perm && p < w) ? perm[p] : p;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3, qbase = lane & ~3;
  auto out_of_range = [](double v) {  // zero, or biased exponent inside [56, 1990]
    const unsigned hi = static_cast<unsigned>(__double_as_longlong(v) >> 32) & 0x7fffffffu;
    const unsigned e = hi >> 20;
    return static_cast<unsigned>((e - 56u) > (1990u - 56u)) & static_cast<unsigned>(v != 0.0);
  };
  for (int64_t tile = blockIdx.x; tile * 64 < M; tile += gridDim.x) {
    const int64_t r0 = tile * 64 + warp * 16 + g;  // rows r0, r0 + 8
    double x[NT][4];  // x[P][v0 + 2 v1] = X(r0 + 8 v1, 8P + 2t + v0)
#pragma unroll
    for (int P = 0; P < NT; ++P)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int q = 8 * P + 2 * t + (v & 1);
        const int64_t j = r0 + 8 * (v >> 1);
        x[P][v] = (q < w && j < M) ? X[j + sperm[q] * ldx] : 0.0;
      }
    // forward: Lhat y = u (unit lower)
#pragma unroll
    for (int P = 0; P < NT; ++P) {
#pragma unroll
      for (int Q = 0; Q < P; ++Q) {
        const double2 b = *reinterpret_cast<const double2*>(sneg + (8 * P + g) * WP + 8 * Q + 2 * t);
        dmma_16x8x8(x[P], x[Q][0], x[Q][2], x[Q][1], x[Q][3], b.x, b.y);
      }
#pragma unroll
      for (int pp = 0; pp < 7; ++pp) {
        const double y0 = __shfl_sync(0xffffffffu, x[P][pp & 1], qbase | (pp >> 1));
        const double y1 = __shfl_sync(0xffffffffu, x[P][2 + (pp & 1)], qbase | (pp >> 1));
#pragma unroll
        for (int dq = 0; dq < 2; ++dq)
          if (2 * t + dq > pp) {
            const double l = sneg[(8 * P + 2 * t + dq) * WP + 8 * P + pp];
            x[P][dq] = fma(l, y0, x[P][dq]);
            x[P][2 + dq] = fma(l, y1, x[P][2 + dq]);
          }
      }
    }
    // back: Uhat x = y
#pragma unroll
    for (int P = NT - 1; P >= 0; --P) {
#pragma unroll
      for (int Q = NT - 1; Q > P; --Q) {
        const double2 b = *reinterpret_cast<const double2*>(sneg + (8 * P + g) * WP + 8 * Q + 2 * t);
        dmma_16x8x8(x[P], x[Q][0], x[Q][2], x[Q][1], x[Q][3], b.x, b.y);
      }
#pragma unroll
      for (int pp = 7; pp >= 0; --pp) {
        const int p = 8 * P + pp;
        const double upp = -sneg[p * WP + p], yr = srcp[p];
        const double a0 = __shfl_sync(0xffffffffu, x[P][pp & 1], qbase | (pp >> 1));
        const double a1 = __shfl_sync(0xffffffffu, x[P][2 + (pp & 1)], qbase | (pp >> 1));
        double x0 = __dmul_rn(a0, yr), x1 = __dmul_rn(a1, yr);
        x0 = __fma_rn(__fma_rn(-x0, upp, a0), yr, x0);
        x1 = __fma_rn(__fma_rn(-x1, upp, a1), yr, x1);
        const unsigned bad = out_of_range(a0) | out_of_range(a1) | out_of_range(x0) | out_of_range(x1) |
                             static_cast<unsigned>(!pivot_in_range(upp));
        if (__any_sync(0xffffffffu, bad)) {
          x0 = ieee_div(a0, upp);
          x1 = ieee_div(a1, upp);
        }
        if (t == (pp >> 1)) {
          x[P][pp & 1] = x0;
          x[P][2 + (pp & 1)] = x1;
        }
#pragma unroll
        for (int dq = 0; dq < 2; ++dq)
          if (2 * t + dq < pp) {
            const double u = sneg[(8 * P + 2 * t + dq) * WP + p];
            x[P][dq] = fma(u, x0, x[P][dq]);
            x[P][2 + dq] = fma(u, x1, x[P][2 + dq]);
          }
      }
    }
#pragma unroll
    for (int P = 0; P < NT; ++P)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int q = 8 * P + 2 * t + (v & 1);
        const int64_t j = r0 + 8 * (v >> 1);
        if (q < w && j < M) out[j + q * ldo] = x[P][v];
      }
  }
}

// Blocked form (A/B: ITERCUR_ROWS_SOLVE_BLK=1): the row in shared memory in chunks of 8 entries, the
// factors zero-padded to 64 x 64. Each chunk of 8 unknowns is updated by every earlier (forward) /
// later (back) chunk with an unrolled 8 x 8 block of FMAs on registers — eight shared-memory reads
// of x per 64 FMAs instead of one per FMA (the per-FMA form above is bound by shared-memory
// bandwidth: 187 us at 100000 x 50). The forward sweep accumulates each x[q] in ascending p like the
// row form; the back sweep subtracts the later chunks before the chunk's own triangle.
__global__ void __launch_bounds__(128) rows_lu_solve_blk_kernel(const double* __restrict__ X, int64_t ldx, int64_t M,
                                                                const double* __restrict__ lu, int64_t ldd,
                                                                const int* __restrict__ d_w, int w_max,
                                                                double* __restrict__ out, int64_t ldo,
                                                                const IterCtl* __restrict__ ctl, int64_t out_off_per_r,
                                                                const int* __restrict__ perm) {
  constexpr int WP = 64, T = 128;
  extern __shared__ double sm[];
  double* slu = sm;             // 64 x 64, zero-padded, ld 64
  double* xs = sm + WP * WP;    // xs[q * 128 + tid]
  __shared__ int sperm[WP];
  griddep_wait();
  griddep_launch_dependents();
  if (ctl) {
    if (ctl->done) return;
    lu += ctl->r * ldd;
    out += ctl->r * out_off_per_r;
    if (perm) perm += ctl->r;
  }
  const int w = d_w ? min(*d_w, w_max) : w_max;
  for (int e = threadIdx.x; e < WP * WP; e += T) {
    const int a = e % WP, b = e / WP;
    slu[e] = (a < w && b < w) ? lu[a + b * ldd] : (a == b ? 1.0 : 0.0);  // identity padding: exact no-ops
  }
  for (int q = threadIdx.x; q < WP; q += T) sperm[q] = (perm && q < w) ? perm[q] : q;
  __syncthreads();
  const int nch = (w + 7) / 8;
  double* x = xs + threadIdx.x;
  for (int64_t j = blockIdx.x * (int64_t)T + threadIdx.x; j < M; j += (int64_t)gridDim.x * T) {
    for (int q = 0; q < nch * 8; ++q) x[q * T] = q < w ? X[j + sperm[q] * ldx] : 0.0;  // P u, zero-padded
    // forward: Lhat y = u (unit lower)
    for (int P = 0; P < nch; ++P) {
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = x[(8 * P + i) * T];
      for (int Q = 0; Q < P; ++Q) {
        double xq[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) xq[k] = x[(8 * Q + k) * T];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double* l = slu + 8 * P + (8 * Q + k) * WP;
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = fma(-l[i], xq[k], v[i]);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double* l = slu + 8 * P + (8 * P + k) * WP;
#pragma unroll
        for (int i = k + 1; i < 8; ++i) v[i] = fma(-l[i], v[k], v[i]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) x[(8 * P + i) * T] = v[i];
    }
    // back: Uhat x = y
    for (int P = nch - 1; P >= 0; --P) {
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = x[(8 * P + i) * T];
      for (int Q = P + 1; Q < nch; ++Q) {
        double xq[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) xq[k] = x[(8 * Q + k) * T];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const double* u = slu + 8 * P + (8 * Q + k) * WP;
#pragma unroll
          for (int i = 0; i < 8; ++i) v[i] = fma(-u[i], xq[k], v[i]);
        }
      }
#pragma unroll
      for (int k = 7; k >= 0; --k) {
        v[k] = v[k] / slu[(8 * P + k) * (WP + 1)];
        const double* u = slu + 8 * P + (8 * P + k) * WP;
#pragma unroll
        for (int i = 0; i < k; ++i) v[i] = fma(-u[i], v[k], v[i]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) x[(8 * P + i) * T] = v[i];
    }
    for (int q = 0; q < w; ++q) out[j + q * ldo] = x[q * T];
  }
}

// generic width (w > 64): same solves with x in a column-strided global workspace; the factors
// in shared memory while w*w doubles fit one CTA (w <= 168), else read from global memory
// (L1/L2-resident: every thread walks them in the same order)
template <bool SMEM>
__global__ void rows_lu_solve_wide_kernel(const double* __restrict__ X, int64_t ldx, int64_t M,
                                          const double* __restrict__ lu, int64_t ldd, const int* __restrict__ d_w,
                                          int w_max, double* __restrict__ out, int64_t ldo,
                                          const IterCtl* __restrict__ ctl, int64_t out_off_per_r,
                                          double* __restrict__ scratch, const int* __restrict__ perm) {
  extern __shared__ double slu[];
  if (ctl) {
    if (ctl->done) return;
    lu += ctl->r * ldd;
    out += ctl->r * out_off_per_r;
    if (perm) perm += ctl->r;
  }
  const int w = d_w ? min(*d_w, w_max) : w_max;
  if (SMEM) {
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) slu[e] = lu[(e % w) + (e / w) * ldd];
    __syncthreads();
  }
  const int64_t ld = SMEM ? w : ldd;
  const double* f = SMEM ? slu : lu;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < M; j += (int64_t)gridDim.x * blockDim.x) {
    double* x = scratch + j;  // column-strided per-row workspace (ld M)
    for (int q = 0; q < w; ++q) x[q * M] = X[j + (perm ? perm[q] : q) * ldx];
    for (int q = 1; q < w; ++q) {
      double v = x[q * M];
      for (int p = 0; p < q; ++p) v = fma(-f[q + p * ld], x[p * M], v);
      x[q * M] = v;
    }
    for (int q = w - 1; q >= 0; --q) {
      double v = x[q * M];
      for (int p = q + 1; p < w; ++p) v = fma(-f[q + p * ld], x[p * M], v);
      x[q * M] = v / f[q + q * ld];
    }
    for (int q = 0; q < w; ++q) out[j + q * ldo] = x[q * M];
  }
}

cudaError_t launch_rows_lu_solve(const double* X, int64_t ldx, int64_t M, const double* lu, int64_t ldd,
                                 const int* d_w, int w_max, double* out, int64_t ldo, cudaStream_t st,
                                 const IterCtl* ctl, int64_t out_off_per_r, const int* perm) {
  if (M <= 0 || w_max <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(M, 128), 148 * 16));
  const size_t smem = sizeof(double) * static_cast<size_t>(w_max) * w_max;
  if (w_max <= 16) {
    return launch_ex(rows_lu_solve_kernel<16>, dim3(blocks), dim3(128), smem, st, dim3(0, 0, 0), X, ldx, M, lu, ldd, d_w,
                     w_max, out, ldo, ctl, out_off_per_r, perm);
  } else if (w_max <= 64 && !env_flag("ITERCUR_ROWS_SOLVE_ROWFORM") && !env_flag("ITERCUR_ROWS_SOLVE_COLFORM") &&
             !env_flag("ITERCUR_ROWS_SOLVE_SMEM") && !env_flag("ITERCUR_ROWS_SOLVE_BLK")) {
    // tensor-core blocked solve: 64 rows per CTA, persistent over the row tiles
    const int tiles = static_cast<int>(std::min<int64_t>(ceil_div(M, 64), 148 * 8));
    switch ((w_max + 7) / 8) {
      case 3: return launch_ex(rows_lu_solve_mma_kernel<3>, dim3(tiles), dim3(128), 0, st, dim3(0, 0, 0), X, ldx, M, lu,
                               ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
      case 4: return launch_ex(rows_lu_solve_mma_kernel<4>, dim3(tiles), dim3(128), 0, st, dim3(0, 0, 0), X, ldx, M, lu,
                               ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
      case 5: return launch_ex(rows_lu_solve_mma_kernel<5>, dim3(tiles), dim3(128), 0, st, dim3(0, 0, 0), X, ldx, M, lu,
                               ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
      case 6: return launch_ex(rows_lu_solve_mma_kernel<6>, dim3(tiles), dim3(128), 0, st, dim3(0, 0, 0), X, ldx, M, lu,
                               ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
      case 7: return launch_ex(rows_lu_solve_mma_kernel<7>, dim3(tiles), dim3(128), 0, st, dim3(0, 0, 0), X, ldx, M, lu,
                               ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
      default: return launch_ex(rows_lu_solve_mma_kernel<8>, dim3(tiles), dim3(128), 0, st, dim3(0, 0, 0), X, ldx, M,
                                lu, ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
    }
  } else if (w_max <= 64 && env_flag("ITERCUR_ROWS_SOLVE_BLK")) {  // A/B: blocked rows in shared memory
    // blocked, rows in shared memory (default; A/B switches below)
    const size_t smem2 = sizeof(double) * (64 * 64 + 64 * 128);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(rows_lu_solve_blk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem2));
      attr = true;
    }
    return launch_ex(rows_lu_solve_blk_kernel, dim3(blocks), dim3(128), smem2, st, dim3(0, 0, 0), X, ldx, M, lu, ldd,
                     d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
  } else if (w_max <= 64 && env_flag("ITERCUR_ROWS_SOLVE_SMEM")) {  // A/B: per-FMA shared-memory form
    const size_t smem2 = sizeof(double) * (64 * 64 + 64 * 128);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(rows_lu_solve_smem_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem2));
      attr = true;
    }
    return launch_ex(rows_lu_solve_smem_kernel<64>, dim3(blocks), dim3(128), smem2, st, dim3(0, 0, 0), X, ldx, M, lu,
                     ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
  } else if (w_max <= 32 && env_flag("ITERCUR_ROWS_SOLVE_ROWFORM")) {  // A/B: the row-oriented register form
    return launch_ex(rows_lu_solve_kernel<32>, dim3(blocks), dim3(128), smem, st, dim3(0, 0, 0), X, ldx, M, lu, ldd, d_w,
                     w_max, out, ldo, ctl, out_off_per_r, perm);
  } else if (w_max <= 64 && env_flag("ITERCUR_ROWS_SOLVE_ROWFORM")) {
    return launch_ex(rows_lu_solve_kernel<64>, dim3(blocks), dim3(128), smem, st, dim3(0, 0, 0), X, ldx, M, lu, ldd, d_w,
                     w_max, out, ldo, ctl, out_off_per_r, perm);
  } else if (w_max <= 64) {  // A/B: lane pairs, column-oriented (64 rows per 128-thread CTA)
    const int blocks2 = static_cast<int>(std::min<int64_t>(ceil_div(M, 64), 148 * 16));
    if (w_max <= 32)
      return launch_ex(rows_lu_solve_col_kernel<32>, dim3(blocks2), dim3(128), smem, st, dim3(0, 0, 0), X, ldx, M, lu,
                       ldd, d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
    return launch_ex(rows_lu_solve_col_kernel<64>, dim3(blocks2), dim3(128), smem, st, dim3(0, 0, 0), X, ldx, M, lu, ldd,
                     d_w, w_max, out, ldo, ctl, out_off_per_r, perm);
  }
  // per-row workspace: M x w doubles (stream-ordered, freed after the launch)
  double* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), sizeof(double) * M * w_max, st);
  if (e != cudaSuccess) return e;
  constexpr size_t kSmemMax = 227 * 1024;
  if (smem <= kSmemMax) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(rows_lu_solve_wide_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kSmemMax));
      attr = true;
    }
    rows_lu_solve_wide_kernel<true><<<blocks, 128, smem, st>>>(X, ldx, M, lu, ldd, d_w, w_max, out, ldo, ctl,
                                                               out_off_per_r, scratch, perm);
  } else {  // blocks wider than ~168: the factors stay in global memory
    rows_lu_solve_wide_kernel<false><<<blocks, 128, 0, st>>>(X, ldx, M, lu, ldd, d_w, w_max, out, ldo, ctl,
                                                             out_off_per_r, scratch, perm);
  }
  e = cudaGetLastError();
  cudaFreeAsync(scratch, st);
  return e;
}

// Column-sharded engine: this shard's columns of the selected block J_k. For q < ncols with
// j = J_k[q] - goff in [0, cnt): PackA(:, q) = A(:, j), PackR(0:r, q) = R~(0:r, j) (R~ row-major,
// ld ldR), PackY(:, q) = Y(:, j). zero_rest: the other shards' columns are written as zeros, so a
// sum-allreduce over the ranks assembles the block exactly (disjoint contributions + 0).
__global__ void pack_owned_kernel(const IterCtl* __restrict__ ctl, const int* __restrict__ d_ncols,
                                  const int64_t* __restrict__ col_idx, int64_t goff, int64_t cnt,
                                  const double* __restrict__ A, int64_t lda, int64_t m,
                                  const double* __restrict__ Rt, int64_t ldR, const double* __restrict__ Y,
                                  int64_t cp, double* __restrict__ PackA, int64_t ldpa, double* __restrict__ PackR,
                                  int64_t ldpr, double* __restrict__ PackY, int zero_rest) {
  griddep_wait();
  griddep_launch_dependents();
  if (ctl->done) return;
  const int q = blockIdx.y;
  if (q >= *d_ncols) return;
  const int64_t j = col_idx[q] - goff;
  const bool owned = j >= 0 && j < cnt;
  if (!owned && !zero_rest) return;
  const int64_t r = ctl->r;
  const int64_t total = m + r + cp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < m) {
      PackA[e + q * ldpa] = owned ? A[e + j * lda] : 0.0;
    } else if (e < m + r) {
      const int64_t k = e - m;
      PackR[k + q * ldpr] = owned ? Rt[k * ldR + j] : 0.0;
    } else {
      const int64_t h = e - m - r;
      PackY[h + q * cp] = owned ? Y[h + j * cp] : 0.0;
    }
  }
}
cudaError_t launch_pack_owned(const IterCtl* ctl, const int* d_ncols, const int64_t* col_idx, int B, int64_t goff,
                              int64_t cnt, const double* A, int64_t lda, int64_t m, const double* Rt, int64_t ldR,
                              int64_t r_cap, const double* Y, int64_t cp, double* PackA, int64_t ldpa, double* PackR,
                              int64_t ldpr, double* PackY, bool zero_rest, cudaStream_t st) {
  const int bx = static_cast<int>(std::min<int64_t>(ceil_div(m + r_cap + cp, 256), 64));
  return launch_ex(pack_owned_kernel, dim3(std::max(bx, 1), B), dim3(256), 0, st, dim3(0, 0, 0), ctl, d_ncols, col_idx,
                   goff, cnt, A, lda, m, Rt, ldR, Y, cp, PackA, ldpa, PackR, ldpr, PackY, zero_rest ? 1 : 0);
}

// CSR (row_ptr, col_idx, values; proj/src/matrix.cpp:79-104 layout) -> dense column-major
// (the output must be zeroed by the caller); one thread per row.
__global__ void csr_to_dense_kernel(int64_t rows, const int64_t* __restrict__ row_ptr,
                                    const int64_t* __restrict__ col_idx, const double* __restrict__ values,
                                    double* __restrict__ out, int64_t ld) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) out[i + col_idx[p] * ld] = values[p];
}
cudaError_t launch_csr_to_dense(int64_t rows, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                                double* out, int64_t ld, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(rows, 256), 148 * 8));
  csr_to_dense_kernel<<<blocks, 256, 0, st>>>(rows, row_ptr, col_idx, values, out, ld);
  return cudaGetLastError();
}

// Sum `count` partials into *out in a fixed order (one CTA).
__global__ void sum_partials_kernel(const double* __restrict__ p, int64_t count, double* __restrict__ out,
                                    const IterCtl* __restrict__ ctl) {
  __shared__ double red[8];
  if (ctl && ctl->done) return;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += p[i];
  const double b = block_sum<256>(s, red);
  if (threadIdx.x == 0) *out = b;
}
cudaError_t launch_sum_partials(const double* partials, int64_t count, double* d_out, cudaStream_t st,
                                const IterCtl* ctl) {
  sum_partials_kernel<<<1, 256, 0, st>>>(partials, count, d_out, ctl);
  return cudaGetLastError();
}

// Per-block sum of squares over a strided 2D region (rows x cols, ld), then fixed-order sum.
__global__ void sumsq_kernel(const double* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                             double* __restrict__ part) {
  __shared__ double red[8];
  double s = 0.0;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    const double v = x[i + j * ld];
    s = fma(v, v, s);
  }
  const double b = block_sum<256>(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}
cudaError_t launch_sumsq(const double* x, int64_t rows, int64_t cols, int64_t ld, double* partials, int max_parts,
                         double* d_out, cudaStream_t st) {
  const int64_t total = rows * cols;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), max_parts)));
  sumsq_kernel<<<blocks, 256, 0, st>>>(x, rows, cols, ld, partials);
  sum_partials_kernel<<<1, 256, 0, st>>>(partials, blocks, d_out, nullptr);
  return cudaGetLastError();
}

// count of non-finite entries (exact check behind a non-finite ||A||^2)
__global__ void nonfinite_kernel(const double* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                 unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / rows, i = e - j * rows;
    if (!isfinite(x[i + j * ld])) ++c;
  }
  if (c) atomicAdd(count, c);
}
cudaError_t launch_count_nonfinite(const double* x, int64_t rows, int64_t cols, int64_t ld, unsigned long long* d_count,
                                   cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows * cols, 256), 148 * 8)));
  nonfinite_kernel<<<blocks, 256, 0, st>>>(x, rows, cols, ld, d_count);
  return cudaGetLastError();
}

// Iteration start (driver.cpp:87-95).
__global__ void iter_begin_kernel(IterCtl* ctl, IterState* slot) {
  griddep_wait();
  griddep_launch_dependents();
  slot->ncols = slot->nrows = slot->width = 0;
  slot->valid = 0;
  if (ctl->done) {
    ctl->block = 0;
    return;
  }
  if (ctl->r >= ctl->max_rank || ctl->k >= ctl->max_iters) {
    ctl->done = 1;
    ctl->status = 1;  // MaxRank
    ctl->block = 0;
    return;
  }
  slot->valid = 1;
  ctl->block = static_cast<int32_t>(min(static_cast<int64_t>(ctl->b), ctl->max_rank - ctl->r));
}
cudaError_t launch_iter_begin(IterCtl* ctl, IterState* slot, cudaStream_t st) {
  return launch_ex(iter_begin_kernel, dim3(1), dim3(1), 0, st, dim3(0, 0, 0), ctl, slot);
}

__global__ void width_kernel(IterState* slot, const IterCtl* ctl) {
  if (ctl->done) return;
  slot->width = min(slot->ncols, slot->nrows);
}
cudaError_t launch_width(IterState* slot, const IterCtl* ctl, cudaStream_t st) {
  width_kernel<<<1, 1, 0, st>>>(slot, ctl);
  return cudaGetLastError();
}

// Iteration commit (driver.cpp:102-159).
__global__ void commit_kernel(CommitArgs c, const double* __restrict__ y_partials, int64_t y_parts) {
  __shared__ double red[8];
  griddep_wait();
  griddep_launch_dependents();
  if (c.ctl->done) return;
  commit_body<256>(c, y_partials, y_parts, red);
}

cudaError_t launch_commit(IterCtl* ctl, IterState* slot, const IterArrays& arr, int64_t* I_all, int64_t* J_all,
                          uint8_t* row_mask, uint8_t* col_mask, const double* y_partials, int64_t y_parts,
                          cudaStream_t st) {
  CommitArgs c;
  c.ctl = ctl;
  c.slot = slot;
  c.row_idx = arr.row_idx;
  c.col_idx = arr.col_idx;
  c.I_all = I_all;
  c.J_all = J_all;
  c.row_mask = row_mask;
  c.col_mask = col_mask;
  return launch_ex(commit_kernel, dim3(1), dim3(256), 0, st, dim3(0, 0, 0), c, y_partials, y_parts);
}

// a kernel of this translation unit (module), for itercur_preload
const void* module_anchor_misc() { return reinterpret_cast<const void*>(gather_kernel); }

}  // namespace itercur_b200

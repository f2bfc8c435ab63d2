// shard.cu — per-rank building blocks of the column-sharded engine.
//
// With A column-sharded over ranks, the column selection (LUPP on Y^T, proj/src/select.cpp:
// 34-74,121-139) runs over rows of Y^T that live on different GPUs. Each pivot step is then
//   (1) every rank eliminates its own rows with the previous step's pivot row and offers its
//       best candidate for the current column (|value|, runner-up, global index, row tail);
//   (2) the candidates are all-gathered (NCCL) and every rank reduces them in rank order —
//       shards are contiguous column ranges in rank order, so "first maximum in rank order"
//       is the reference's lowest-index tie rule;
// which reproduces the single-device pivot sequence exactly (same per-row operations:
// factor = W(i,s)/pivot, W(i,t) -= factor * W(p,t), two roundings, no FMA).
// The other per-rank pieces are plain building blocks: a dense in-place LU without pivoting
// (the cross block D_k, rows already in pivot order, as cross_lu_kernel in misc.cu).
#include "common.cuh"
#include "kernels.h"

namespace itercur_b200 {

constexpr int kDistThreads = 1024;

// One CTA: the per-step work of one rank is a few thousand rows of a narrow panel.
__global__ void __launch_bounds__(kDistThreads) lupp_dist_step_kernel(double* __restrict__ W, int64_t rows,
                                                                      int64_t ldw, int steps, int s,
                                                                      const double* __restrict__ P, int64_t piv_local,
                                                                      uint8_t* __restrict__ live, int64_t row_offset,
                                                                      double* __restrict__ cand) {
  __shared__ Cand sc[kDistThreads / 32 + 1];
  if (P && piv_local >= 0 && piv_local < rows && threadIdx.x == 0) live[piv_local] = 0;
  __syncthreads();
  Cand mine = cand_empty();
  for (int64_t i = threadIdx.x; i < rows; i += kDistThreads) {
    if (!live[i]) continue;
    if (P) {
      const double f = __ddiv_rn(W[i + (s - 1) * ldw], P[s - 1]);
      for (int t = s; t < steps; ++t) W[i + t * ldw] = __dsub_rn(W[i + t * ldw], __dmul_rn(f, P[t]));
    }
    const double mag = fabs(W[i + s * ldw]);
    // ascending rows per thread: strict '>' keeps the lowest index on ties
    if (mag > mine.mag) {
      mine.second = fmax(mine.second, mine.mag);
      mine.mag = mag;
      mine.idx = row_offset + i;
    } else {
      mine.second = fmax(mine.second, mag);
    }
  }
  mine = warp_reduce_cand(mine);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sc[warp] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand r = sc[0];
    for (int q = 1; q < kDistThreads / 32; ++q) r = cand_merge(r, sc[q]);
    sc[kDistThreads / 32] = r;
    cand[0] = r.idx >= 0 ? r.mag : -1.0;
    cand[1] = r.second;
    cand[2] = static_cast<double>(r.idx);
    cand[3] = 0.0;
  }
  __syncthreads();
  const Cand r = sc[kDistThreads / 32];
  for (int t = threadIdx.x; t < steps; t += kDistThreads)
    cand[4 + t] = (r.idx >= 0 && t >= s) ? W[(r.idx - row_offset) + t * ldw] : 0.0;
}

cudaError_t launch_lupp_dist_step(double* W, int64_t rows, int64_t ldw, int steps, int s, const double* P,
                                  int64_t piv_local, uint8_t* live, int64_t row_offset, double* cand,
                                  cudaStream_t st) {
  lupp_dist_step_kernel<<<1, kDistThreads, 0, st>>>(W, rows, ldw, steps, s, P, piv_local, live, row_offset, cand);
  return cudaGetLastError();
}

// In-place Doolittle LU without pivoting of a w x w block (same operations and order as
// cross_lu_kernel: f = D(p,s)/D(s,s); D(p,q) -= f*D(s,q); then D(p,s) = f).
__global__ void dense_lu_kernel(double* __restrict__ D, int w, int64_t ldd) {
  for (int s = 0; s < w; ++s) {
    const double piv = D[s + s * ldd];
    const int rem = w - s - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      const int p = s + 1 + e % rem, q = s + 1 + e / rem;
      const double f = __ddiv_rn(D[p + s * ldd], piv);
      D[p + q * ldd] = __dsub_rn(D[p + q * ldd], __dmul_rn(f, D[s + q * ldd]));
    }
    __syncthreads();
    for (int p = s + 1 + threadIdx.x; p < w; p += blockDim.x) D[p + s * ldd] = __ddiv_rn(D[p + s * ldd], piv);
    __syncthreads();
  }
}

cudaError_t launch_dense_lu(double* D, int w, int64_t ldd, cudaStream_t st) {
  if (w <= 0) return cudaSuccess;
  dense_lu_kernel<<<1, 256, 0, st>>>(D, w, ldd);
  return cudaGetLastError();
}

// a kernel of this translation unit (module), for itercur_preload
const void* module_anchor_shard() { return reinterpret_cast<const void*>(dense_lu_kernel); }

}  // namespace itercur_b200

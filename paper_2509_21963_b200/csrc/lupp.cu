// lupp.cu — pivot selection by LU with partial pivoting, one persistent cooperative
// kernel per call (proj/src/select.cpp:34-74 lupp_pivot_rows; used for select_columns on
// W = Y^T, select.cpp:121-139, and for select_rows on W = S_row, select.cpp:141-165).
//
// Each step s of the reference is: argmax over unbanned rows of |W(i,s)| (ties -> lowest
// index), the absolute / relative floors, then a rank-1 elimination of the remaining
// rows with factor = W(i,s)/pivot and W(i,t) -= factor * W(best,t) (two roundings, no FMA).
// Here every CTA owns a fixed strided set of rows for the whole call; per step it
// eliminates its rows, computes its local (max, lowest index, runner-up) candidate on
// column s+1 in the same pass, publishes it, and one grid-wide barrier later every CTA
// reduces the same candidate list in the same order — so the pivot sequence is exactly
// the reference's for identical W bits. Only the columns that can still become a pivot
// column (t < steps) are eliminated; the reference also updates columns >= steps, which
// are never read again.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace itercur_b200 {

constexpr int kLuppThreads = 256;

__device__ __forceinline__ Cand block_reduce_cand(Cand c, Cand* sc) {
  c = warp_reduce_cand(c);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sc[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand r = sc[0];
    for (int w = 1; w < kLuppThreads / 32; ++w) r = cand_merge(r, sc[w]);
    sc[kLuppThreads / 32] = r;
  }
  __syncthreads();
  Cand r = sc[kLuppThreads / 32];
  __syncthreads();
  return r;
}

struct LuppKernelArgs {
  LuppArgs a;
  Cand* cand;           // [2][gridDim.x]
  double* norm_part;    // [gridDim.x]
};

__global__ void __launch_bounds__(kLuppThreads) lupp_kernel(LuppKernelArgs ka) {
  cg::grid_group grid = cg::this_grid();
  const LuppArgs& a = ka.a;
  extern __shared__ double prow[];  // pivot-row tail, cols_max doubles
  __shared__ Cand sc[kLuppThreads / 32 + 1];
  __shared__ double sred[kLuppThreads / 32];

  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * kLuppThreads + threadIdx.x;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * kLuppThreads;
  const int G = gridDim.x;
  const uint8_t ep = a.epoch;
  double* W = a.W;
  const int64_t ldw = a.ldw;
  int steps = a.cols_max;
  if (a.d_steps) steps = min(steps, *a.d_steps);
  if (steps <= 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_count = 0;
    return;
  }

  // ---- absolute floor 100 * eps * ||M||_F (select.cpp:11,127,144) ----
  double nsq;
  if (a.d_norm_sq) {
    nsq = *a.d_norm_sq;
  } else {
    double s = 0.0;
    for (int t = 0; t < steps; ++t)
      for (int64_t i = gtid; i < a.rows; i += gstride) {
        const double v = W[i + t * ldw];
        s = fma(v, v, s);
      }
    const double b = block_sum<kLuppThreads>(s, sred);
    if (threadIdx.x == 0) ka.norm_part[blockIdx.x] = b;
    grid.sync();
    nsq = 0.0;
    for (int q = 0; q < G; ++q) nsq += ka.norm_part[q];
  }
  const double abs_floor = 1e2 * 2.220446049250313e-16 * sqrt(nsq);

  // ---- step-0 candidates ----
  Cand local = cand_empty();
  for (int64_t i = gtid; i < a.rows; i += gstride) {
    const uint8_t mk = a.mask[i];
    if (mk == 1 || mk == ep) continue;
    local = cand_merge(local, Cand{fabs(W[i]), -1.0, i});
  }
  Cand bc = block_reduce_cand(local, sc);
  if (threadIdx.x == 0) ka.cand[blockIdx.x] = bc;
  grid.sync();

  int count = 0;
  double first = 0.0;
  for (int s = 0; s < steps; ++s) {
    // every CTA reduces the same list in the same order
    const Cand* cs = ka.cand + (s & 1) * G;
    Cand r = cand_empty();
    for (int q = threadIdx.x; q < G; q += kLuppThreads) r = cand_merge(r, cs[q]);
    const Cand best = block_reduce_cand(r, sc);
    if (best.idx < 0 || best.mag <= abs_floor) break;
    if (s == 0)
      first = best.mag;
    else if (best.mag < a.pivot_floor * first)
      break;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.d_idx[s] = best.idx;
      a.d_best[s] = best.mag;
      a.d_second[s] = best.second;
    }
    ++count;
    if (s + 1 >= steps) break;

    const double pivot = W[best.idx + s * ldw];
    for (int t = s + 1 + threadIdx.x; t < steps; t += kLuppThreads) prow[t] = W[best.idx + t * ldw];
    __syncthreads();
    local = cand_empty();
    for (int64_t i = gtid; i < a.rows; i += gstride) {
      if (i == best.idx) {
        a.mask[i] = ep;
        continue;
      }
      const uint8_t mk = a.mask[i];
      if (mk == 1 || mk == ep) continue;
      const double f = __ddiv_rn(W[i + s * ldw], pivot);
      double nxt = 0.0;
      for (int t = s + 1; t < steps; ++t) {
        const double v = __dsub_rn(W[i + t * ldw], __dmul_rn(f, prow[t]));
        W[i + t * ldw] = v;
        if (t == s + 1) nxt = v;
      }
      local = cand_merge(local, Cand{fabs(nxt), -1.0, i});
    }
    bc = block_reduce_cand(local, sc);
    if (threadIdx.x == 0) ka.cand[((s + 1) & 1) * G + blockIdx.x] = bc;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.d_count = count;
}

// Clear in-call ban marks (any value other than 1) when the epoch counter wraps.
__global__ void clear_epochs_kernel(uint8_t* mask, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    if (mask[i] != 1) mask[i] = 0;
}

cudaError_t launch_clear_epochs(uint8_t* mask, int64_t count, cudaStream_t st) {
  const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(count, 256), 1184));
  clear_epochs_kernel<<<std::max(blocks, 1), 256, 0, st>>>(mask, count);
  return cudaGetLastError();
}

static int lupp_max_blocks() {
  static int max_blocks = -1;
  if (max_blocks < 0) {
    int per_sm = 0;
    cudaFuncSetAttribute(lupp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lupp_kernel, kLuppThreads, 16 * 1024);
    int dev = 0, sms = kNumSMs;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    max_blocks = std::max(1, per_sm) * sms;
  }
  return max_blocks;
}

// scratch: caller-provided device buffer of >= lupp_scratch_bytes() bytes
size_t lupp_scratch_bytes() { return sizeof(Cand) * 2 * 4096 + sizeof(double) * 4096; }

cudaError_t run_lupp_with_scratch(const LuppArgs& a, void* scratch, cudaStream_t st, int* grid_used) {
  if (a.cols_max > 2048) return cudaErrorInvalidValue;
  const int64_t want = std::max<int64_t>(1, ceil_div(a.rows, kLuppThreads * 4));
  int grid = static_cast<int>(std::min<int64_t>(want, std::min(lupp_max_blocks(), 4096)));
  LuppKernelArgs ka;
  ka.a = a;
  ka.cand = reinterpret_cast<Cand*>(scratch);
  ka.norm_part = reinterpret_cast<double*>(reinterpret_cast<char*>(scratch) + sizeof(Cand) * 2 * 4096);
  void* params[] = {&ka};
  const size_t smem = sizeof(double) * std::max(a.cols_max, 1);
  if (grid_used) *grid_used = grid;
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lupp_kernel), dim3(grid), dim3(kLuppThreads),
                                     params, smem, st);
}

}  // namespace itercur_b200

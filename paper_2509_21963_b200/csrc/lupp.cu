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
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.d_count = 0;
      if (a.d_width_out) *a.d_width_out = 0;
    }
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
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
  }
}

// ---------------------------------------------------------------------------------
// Shared-memory-resident variant (used whenever a CTA's rows x steps slab fits): every CTA
// loads its contiguous slab of W once, eliminates it in shared memory, and publishes per
// step its candidate (|W(i,s+1)|, index, runner-up) together with that row's remaining
// entries, so after the grid barrier every CTA has the winning pivot row without another
// round trip. Per step: one grid barrier, G candidates read, R_b x (steps-s-1) shared updates
// spread over all threads. Same arithmetic (and therefore the same pivots) as above.
// ---------------------------------------------------------------------------------
struct LuppSmemArgs {
  LuppArgs a;
  double* pub;        // [2][G][pub_stride]: mag, second, idx, then the row tail
  int pub_stride;
  double* norm_part;  // [G]
  int rows_per_cta;
};

__global__ void __launch_bounds__(kLuppThreads) lupp_smem_kernel(LuppSmemArgs ka) {
  cg::grid_group grid = cg::this_grid();
  const LuppArgs& a = ka.a;
  extern __shared__ double sm[];
  __shared__ Cand sc[kLuppThreads / 32 + 1];
  __shared__ double sred[kLuppThreads / 32];
  __shared__ int s_winner;
  const int G = gridDim.x;
  const int Rb = ka.rows_per_cta;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * Rb;
  int64_t nr64 = a.rows - r0;
  nr64 = nr64 < 0 ? 0 : (nr64 > Rb ? Rb : nr64);
  const int nr = static_cast<int>(nr64);
  int steps = a.cols_max;
  if (a.d_steps) steps = min(steps, *a.d_steps);
  if (steps <= 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.d_count = 0;
      if (a.d_width_out) *a.d_width_out = 0;
    }
    return;
  }
  double* Ws = sm;                                   // [steps][Rb]
  double* F = Ws + static_cast<size_t>(steps) * Rb;  // [Rb] elimination factors
  double* prow = F + Rb;                             // [steps]
  uint8_t* banned = reinterpret_cast<uint8_t*>(prow + steps);  // [Rb]

  for (int e = threadIdx.x; e < steps * nr; e += kLuppThreads) {
    const int t = e / nr, r = e - t * nr;
    Ws[t * Rb + r] = a.W[(r0 + r) + t * a.ldw];
  }
  for (int r = threadIdx.x; r < nr; r += kLuppThreads) {
    const uint8_t mk = a.mask[r0 + r];
    banned[r] = (mk == 1 || mk == a.epoch) ? 1 : 0;
  }
  __syncthreads();

  double nsq;
  if (a.d_norm_sq) {
    nsq = *a.d_norm_sq;
  } else {
    double sq = 0.0;
    for (int e = threadIdx.x; e < steps * nr; e += kLuppThreads) {
      const int t = e / nr, r = e - t * nr;
      const double v = Ws[t * Rb + r];
      sq = fma(v, v, sq);
    }
    const double b = block_sum<kLuppThreads>(sq, sred);
    if (threadIdx.x == 0) ka.norm_part[blockIdx.x] = b;
    grid.sync();
    nsq = 0.0;
    for (int q = 0; q < G; ++q) nsq += ka.norm_part[q];
  }
  const double abs_floor = 1e2 * 2.220446049250313e-16 * sqrt(nsq);

  // publish this CTA's candidate on column `col` (and its row tail from `col`)
  auto publish = [&](int col, int parity) {
    Cand local = cand_empty();
    for (int r = threadIdx.x; r < nr; r += kLuppThreads)
      if (!banned[r]) local = cand_merge(local, Cand{fabs(Ws[col * Rb + r]), -1.0, r0 + r});
    const Cand bc = block_reduce_cand(local, sc);
    double* slot = ka.pub + (static_cast<size_t>(parity) * G + blockIdx.x) * ka.pub_stride;
    if (threadIdx.x == 0) {
      slot[0] = bc.mag;
      slot[1] = bc.second;
      slot[2] = __longlong_as_double(bc.idx);
    }
    if (bc.idx >= 0) {
      const int lr = static_cast<int>(bc.idx - r0);
      for (int t = col + threadIdx.x; t < steps; t += kLuppThreads) slot[3 + t] = Ws[t * Rb + lr];
    }
  };

  publish(0, 0);
  grid.sync();
  int count = 0;
  double first = 0.0;
  for (int s = 0; s < steps; ++s) {
    const double* pubs = ka.pub + static_cast<size_t>(s & 1) * G * ka.pub_stride;
    Cand r = cand_empty();
    for (int q = threadIdx.x; q < G; q += kLuppThreads) {
      const double* slot = pubs + static_cast<size_t>(q) * ka.pub_stride;
      r = cand_merge(r, Cand{slot[0], slot[1], __double_as_longlong(slot[2])});
    }
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
    // winner CTA = the one whose published index is best.idx (rows are CTA-contiguous)
    if (threadIdx.x == 0) s_winner = static_cast<int>(best.idx / Rb);
    __syncthreads();
    const double* wslot = pubs + static_cast<size_t>(s_winner) * ka.pub_stride;
    for (int t = s + threadIdx.x; t < steps; t += kLuppThreads) prow[t] = wslot[3 + t];
    if (best.idx >= r0 && best.idx < r0 + nr && threadIdx.x == 0) banned[best.idx - r0] = 1;
    __syncthreads();
    const double pivot = prow[s];
    for (int rr = threadIdx.x; rr < nr; rr += kLuppThreads)
      F[rr] = banned[rr] ? 0.0 : __ddiv_rn(Ws[s * Rb + rr], pivot);
    __syncthreads();
    const int ncols = steps - s - 1;
    for (int e = threadIdx.x; e < ncols * nr; e += kLuppThreads) {
      const int t = s + 1 + e / nr, rr = e - (e / nr) * nr;
      if (!banned[rr]) Ws[t * Rb + rr] = __dsub_rn(Ws[t * Rb + rr], __dmul_rn(F[rr], prow[t]));
    }
    __syncthreads();
    publish(s + 1, (s + 1) & 1);
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
  }
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

static int lupp_max_blocks(const void* fn, size_t smem) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kLuppThreads, smem);
  int dev = 0, sms = kNumSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(0, per_sm) * sms;
}

constexpr int kMaxLuppGrid = 1024;
constexpr size_t kLuppSmemBudget = 200 * 1024;

// scratch: caller-provided device buffer of >= lupp_scratch_bytes(b) bytes
size_t lupp_scratch_bytes(int b) {
  return sizeof(Cand) * 2 * kMaxLuppGrid + sizeof(double) * kMaxLuppGrid +
         sizeof(double) * 2 * kMaxLuppGrid * static_cast<size_t>(b + 4);
}

cudaError_t run_lupp_with_scratch(const LuppArgs& a, void* scratch, cudaStream_t st, int* grid_used) {
  if (a.cols_max > 2048) return cudaErrorInvalidValue;
  char* sp = reinterpret_cast<char*>(scratch);
  Cand* cand = reinterpret_cast<Cand*>(sp);
  double* norm_part = reinterpret_cast<double*>(sp + sizeof(Cand) * 2 * kMaxLuppGrid);
  double* pub = norm_part + kMaxLuppGrid;
  const int steps = std::max(a.cols_max, 1);
  // shared-memory-resident path: one CTA per SM, slab of rows_per_cta x steps doubles
  {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int G = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sms, ceil_div(a.rows, 32))));
    const int Rb = static_cast<int>(ceil_div(a.rows, G));
    const size_t smem = sizeof(double) * (static_cast<size_t>(steps) * Rb + Rb + steps) + Rb + 16;
    if (smem <= kLuppSmemBudget) {
      static size_t attr = 0;
      if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(lupp_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kLuppSmemBudget));
        if (e != cudaSuccess) return e;
        attr = kLuppSmemBudget;
      }
      if (lupp_max_blocks(reinterpret_cast<const void*>(lupp_smem_kernel), smem) >= G) {
        LuppSmemArgs ka;
        ka.a = a;
        ka.pub = pub;
        ka.pub_stride = steps + 3;
        ka.norm_part = norm_part;
        ka.rows_per_cta = Rb;
        void* params[] = {&ka};
        if (grid_used) *grid_used = G;
        return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lupp_smem_kernel), dim3(G),
                                           dim3(kLuppThreads), params, smem, st);
      }
    }
  }
  // global-memory path (slab too large for shared memory)
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(lupp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
    attr_set = true;
  }
  const size_t smem = sizeof(double) * static_cast<size_t>(steps);
  const int64_t want = std::max<int64_t>(1, ceil_div(a.rows, kLuppThreads * 4));
  const int maxb = lupp_max_blocks(reinterpret_cast<const void*>(lupp_kernel), smem);
  int grid = static_cast<int>(std::min<int64_t>(want, std::min(maxb, kMaxLuppGrid)));
  LuppKernelArgs ka;
  ka.a = a;
  ka.cand = cand;
  ka.norm_part = norm_part;
  void* params[] = {&ka};
  if (grid_used) *grid_used = grid;
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lupp_kernel), dim3(grid), dim3(kLuppThreads),
                                     params, smem, st);
}

}  // namespace itercur_b200

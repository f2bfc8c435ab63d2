// qrcp.cu — greedy orthogonalised-column-norm pivoting (QRCP selection), the reference's
// alternative to LUPP: proj/src/select.cpp:79-117 qrcp_pivot_cols, used by select_columns
// (candidates = columns of Y, select.cpp:121-139) and select_rows (candidates = rows of
// S_row, select.cpp:141-165) when col_method / row_method = "qrcp".
//
// Per step: the squared norms of all live candidates (recomputed from the updated
// candidates, as the reference does), the global argmax (strictly greater, so the lowest
// index wins ties), the floors, then q = W(:,best)/|best| and every live candidate loses its
// component along q: w -= q (q . w). One cooperative grid, one candidate per thread
// (grid-stride), one grid barrier per step; each thread folds the next step's norm into its
// update pass. Sums run sequentially over the candidate's entries with separately rounded
// multiply and add — the oracle's order — so the pivots match it bit for bit on equal
// input bits.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "misc.h"

namespace cg = cooperative_groups;

namespace itercur_b200 {

constexpr int kQrcpThreads = 256;
constexpr int kQrcpMaxLen = 256;  // candidate length (sketch rows c or block width w)

struct QrcpArgs {
  double* W;            // candidate j, entry i at W[i * rs + j * cs]
  int64_t ncand;
  int len;              // candidate length (host bound) ...
  const int* d_len;     // ... optionally capped on the device (the row selection's |J_k|)
  int64_t rs, cs;
  const int* d_steps;   // requested steps (device), capped by min(len, ncand)
  int steps_max;
  uint8_t* mask;        // 1 = excluded / already selected (ban marks of the caller)
  uint8_t epoch;        // in-call ban mark (cleared by the caller's epoch protocol)
  const double* d_norm_sq;  // ||M||_F^2 for the absolute floor; nullptr: computed here
  double* norm_part;        // [gridDim.x] scratch for that reduction
  double pivot_floor;
  int64_t* d_idx;
  double* d_best;
  double* d_second;
  int* d_count;
  int* d_width_out;
  const int* d_width_cap;
  Cand* cand;           // [2][gridDim.x] per-CTA candidates (scratch)
  const IterCtl* ctl;   // optional: skip when the run is done
};

__device__ __forceinline__ double cand_sq(const double* w, int len, int64_t rs) {
  double sq = 0.0;
  for (int i = 0; i < len; ++i) sq = __dadd_rn(sq, __dmul_rn(w[i * rs], w[i * rs]));
  return sq;
}

__global__ void __launch_bounds__(kQrcpThreads) qrcp_kernel(QrcpArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Cand sc[kQrcpThreads / 32 + 1];
  __shared__ double q[kQrcpMaxLen];
  __shared__ Cand s_win;
  if (a.ctl && a.ctl->done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.d_count = 0;
      if (a.d_width_out) *a.d_width_out = 0;
    }
    return;  // uniform over the grid
  }
  const int len = a.d_len ? min(a.len, *a.d_len) : a.len;
  int steps = a.steps_max;
  if (a.d_steps) steps = min(steps, *a.d_steps);
  steps = min(steps, len);
  steps = static_cast<int>(min(static_cast<int64_t>(steps), a.ncand));
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kQrcpThreads;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kQrcpThreads + threadIdx.x;
  double nsq;
  if (a.d_norm_sq) {
    nsq = *a.d_norm_sq;
  } else {  // ||M||_F^2 over every candidate (select.cpp:127,145), fixed-order two-level sum
    double sq = 0.0;
    for (int64_t j = j0; j < a.ncand; j += stride)
      for (int i = 0; i < len; ++i) sq = fma(a.W[i * a.rs + j * a.cs], a.W[i * a.rs + j * a.cs], sq);
    __shared__ double red[kQrcpThreads / 32];
    const double b = block_sum<kQrcpThreads>(sq, red);
    if (threadIdx.x == 0) a.norm_part[blockIdx.x] = b;
    grid.sync();
    nsq = 0.0;
    for (unsigned q = 0; q < gridDim.x; ++q) nsq += a.norm_part[q];
  }
  const double abs_floor = 1e2 * 2.220446049250313e-16 * sqrt(nsq);
  // this thread's candidates are j0 + k*stride; bit k of `sel` = selected in this call
  uint32_t sel = 0;
  auto live = [&](int64_t j, int k) {
    const uint8_t mk = a.mask[j];
    return !(mk == 1 || mk == a.epoch) && !(sel >> k & 1u);
  };

  // squared norms of this thread's candidates for step 0
  Cand mine = cand_empty();
  {
    int k = 0;
    for (int64_t j = j0; j < a.ncand; j += stride, ++k)
      if (live(j, k)) {
        const double sq = cand_sq(a.W + j * a.cs, len, a.rs);
        if (sq > mine.mag) mine = Cand{sq, -1.0, j};  // ascending j per thread: strict '>' keeps the lowest
      }
  }
  int count = 0;
  double first = 0.0;
  for (int s = 0; s < steps; ++s) {
    // CTA candidate -> global, then every CTA reduces all CTA candidates in the same order
    Cand c = warp_reduce_cand(mine);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sc[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      Cand r = sc[0];
      for (int w = 1; w < kQrcpThreads / 32; ++w) r = cand_merge(r, sc[w]);
      a.cand[(s & 1) * gridDim.x + blockIdx.x] = r;
    }
    grid.sync();
    if (threadIdx.x == 0) {
      Cand r = a.cand[(s & 1) * gridDim.x];
      for (unsigned b = 1; b < gridDim.x; ++b) r = cand_merge(r, a.cand[(s & 1) * gridDim.x + b]);
      s_win = r;
    }
    __syncthreads();
    const Cand win = s_win;
    if (win.idx < 0) break;
    const double best_mag = sqrt(win.mag);
    if (best_mag <= abs_floor) break;
    if (s == 0)
      first = best_mag;
    else if (best_mag < a.pivot_floor * first)
      break;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.d_idx[s] = win.idx;
      a.d_best[s] = best_mag;
      a.d_second[s] = -1.0;  // QRCP keeps no runner-up (no margin log, as the oracle)
    }
    ++count;
    // q = W(:, best) / |best| (every CTA; the winner column is frozen from now on)
    for (int i = threadIdx.x; i < len; i += kQrcpThreads) q[i] = __ddiv_rn(a.W[i * a.rs + win.idx * a.cs], best_mag);
    __syncthreads();
    // project q out of every live candidate; the next step's norms on the way
    mine = cand_empty();
    if (j0 <= win.idx && (win.idx - j0) % stride == 0) sel |= 1u << ((win.idx - j0) / stride);
    int k = 0;
    for (int64_t j = j0; j < a.ncand; j += stride, ++k) {
      if (!live(j, k)) continue;
      double* w = a.W + j * a.cs;
      double dot = 0.0;
      for (int i = 0; i < len; ++i) dot = __dadd_rn(dot, __dmul_rn(q[i], w[i * a.rs]));
      for (int i = 0; i < len; ++i) w[i * a.rs] = __dsub_rn(w[i * a.rs], __dmul_rn(q[i], dot));
      const double sq = cand_sq(w, len, a.rs);
      if (sq > mine.mag) mine = Cand{sq, -1.0, j};
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
  }
}

size_t qrcp_scratch_bytes() { return sizeof(Cand) * 2 * 1184 + sizeof(double) * 1184; }

cudaError_t run_qrcp(double* W, int64_t ncand, int len, const int* d_len, int64_t rs, int64_t cs, const int* d_steps,
                     int steps_max,
                     uint8_t* mask, uint8_t epoch, const double* d_norm_sq, double pivot_floor, int64_t* d_idx,
                     double* d_best, double* d_second, int* d_count, int* d_width_out, const int* d_width_cap,
                     void* scratch, const IterCtl* ctl, cudaStream_t st) {
  if (len > kQrcpMaxLen || ncand > 32ll * 1184 * kQrcpThreads) return cudaErrorInvalidValue;
  QrcpArgs a;
  a.W = W;
  a.ncand = ncand;
  a.len = len;
  a.d_len = d_len;
  a.rs = rs;
  a.cs = cs;
  a.d_steps = d_steps;
  a.steps_max = steps_max;
  a.mask = mask;
  a.epoch = epoch;
  a.d_norm_sq = d_norm_sq;
  a.pivot_floor = pivot_floor;
  a.d_idx = d_idx;
  a.d_best = d_best;
  a.d_second = d_second;
  a.d_count = d_count;
  a.d_width_out = d_width_out;
  a.d_width_cap = d_width_cap;
  a.cand = static_cast<Cand*>(scratch);
  a.norm_part = reinterpret_cast<double*>(static_cast<char*>(scratch) + sizeof(Cand) * 2 * 1184);
  a.ctl = ctl;
  static int max_blocks = 0;
  if (!max_blocks) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrcp_kernel, kQrcpThreads, 0);
    max_blocks = std::max(1, std::min(per_sm * kNumSMs, 1184));
  }
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_blocks, ceil_div(ncand, kQrcpThreads))));
  void* params[] = {&a};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(qrcp_kernel), dim3(grid), dim3(kQrcpThreads),
                                     params, 0, st);
}

// a kernel of this translation unit (module), for itercur_preload
const void* module_anchor_qrcp() { return reinterpret_cast<const void*>(qrcp_kernel); }

}  // namespace itercur_b200

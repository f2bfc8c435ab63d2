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
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "misc.h"

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

// Warp-level exact argmax with the reference's tie rule, built on redux.sync: a candidate
// is key = bits(|w|) + 1 (0 = none; non-negative doubles order like their bit patterns),
// the winner is the largest key, ties -> lowest row index. `second` is the largest
// magnitude among all other candidates (runner-up, for the margin log).
struct WCand {
  uint64_t key;
  int32_t idx;     // row index (< 2^31 on this path)
  double second;   // -1 if none
};
__device__ __forceinline__ uint64_t mag_key(double mag) {
  return static_cast<uint64_t>(__double_as_longlong(mag)) + 1ull;
}
__device__ __forceinline__ double key_mag(uint64_t key) {
  return key ? __longlong_as_double(static_cast<long long>(key - 1ull)) : -1.0;
}
#ifdef ITERCUR_ARGMAX_SHFL
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__device__ __forceinline__ int warp_min_i32(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
#else
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}
__device__ __forceinline__ int warp_min_i32(int v) { return __reduce_min_sync(0xffffffffu, v); }
#endif
__device__ __forceinline__ WCand warp_argmax(const WCand& c) {
  const uint64_t best = warp_max_u64(c.key);
  const int32_t tie_idx = (c.key == best && best != 0) ? c.idx : 0x7fffffff;
  const int32_t widx = warp_min_i32(tie_idx);
  const bool winner = best != 0 && c.key == best && c.idx == widx;
  // runner-up: the winner lane offers its own second, every other lane its best
  const double offer = winner ? c.second : key_mag(c.key);
  const uint64_t okey = offer >= 0.0 ? mag_key(offer) : 0ull;
  const uint64_t sec = warp_max_u64(okey);
  WCand r;
  r.key = best;
  r.idx = best ? widx : -1;
  r.second = key_mag(sec);
  return r;
}
__device__ __forceinline__ WCand wcand_merge_row(WCand c, double mag, int32_t idx) {
  // sequential scan in ascending row order: strict '>' keeps the lowest index on ties
  const uint64_t k = mag_key(mag);
  if (k > c.key) {
    c.second = key_mag(c.key);
    c.key = k;
    c.idx = idx;
  } else if (mag > c.second) {
    c.second = mag;
  }
  return c;
}

struct LuppKernelArgs {
  LuppArgs a;
  Cand* cand;           // [2][gridDim.x]
  double* norm_part;    // [gridDim.x]
  long long* dbg;       // optional per-step clock64() trace of CTA 0 (panel kernel; benchmarking)
  unsigned long long* arrivals = nullptr;  // panel kernel: monotonic count of published CTA candidates
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
      // columns in chunks of 8: all loads of a chunk are issued before its stores, so the
      // L2 round trips overlap instead of serialising on the possible aliasing
      for (int t0 = s + 1; t0 < steps; t0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = (t0 + u < steps) ? W[i + (t0 + u) * ldw] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (t0 + u < steps) {
            v[u] = __dsub_rn(v[u], __dmul_rn(f, prow[t0 + u]));
            W[i + (t0 + u) * ldw] = v[u];
          }
        }
        if (t0 == s + 1) nxt = v[0];
      }
      local = cand_merge(local, Cand{fabs(nxt), -1.0, i});
    }
    bc = block_reduce_cand(local, sc);
    if (threadIdx.x == 0) ka.cand[((s + 1) & 1) * G + blockIdx.x] = bc;
    grid.sync();
  }
  if (blockIdx.x == 0) {
    // drop this call's in-call ban marks (pivots) so the next call may reuse the same epoch;
    // no CTA reads the mask after the final pivot decision
    __syncthreads();  // d_idx was written by thread 0
    for (int q = threadIdx.x; q < count; q += kLuppThreads) {
      const int64_t i = a.d_idx[q];
      if (a.mask[i] == ep) a.mask[i] = 0;
    }
    if (threadIdx.x == 0) {
      *a.d_count = count;
      if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
    }
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
  double* pub;        // [2][G][pub_stride]: tag, mag, second, idx, then the row tail
  int pub_stride;
  double* norm_part;  // [G]
  int rows_per_cta;
  uint32_t gen;       // per-call generation: slot tags are (gen << 32) | (step + 1)
};

__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Pipelined per-CTA schedule. Warp 0 is the communication warp (owns no rows); warps 1..7
// own the CTA's rows. Per pivot step s:
//   compute warps: read the pivot (s_best / prow of step s), eliminate only column s+1 of
//     their rows (factor = W(i,s)/pivot, kept for later), take the candidate on column s+1,
//     and each warp materialises its own winner row's tail (columns >= s+2) from the
//     not-yet-updated values; [B2]; then apply the deferred updates of columns >= s+2 —
//     overlapped with the exchange below.
//   warp 0: [B2]; block argmax over the warps; write the CTA slot (header + tail) and
//     release it with a (generation, step) tag; poll the G tags with acquire loads — the
//     arrivals are the barrier; read the headers, reduce them in the same order as every
//     other CTA, fetch the winner's tail; publish s_best / prow of step s+1 (double-buffered).
//   [B1] all threads.
// The arithmetic per element is the reference's (factor = W(i,s)/pivot, W(i,t) -= factor *
// W(best,t), separate roundings), so the pivot sequence is identical to select.cpp:40-70.
constexpr int kCompWarps = kLuppThreads / 32 - 1;

__global__ void __launch_bounds__(kLuppThreads) lupp_smem_kernel(LuppSmemArgs ka) {
  cg::grid_group grid = cg::this_grid();
  const LuppArgs& a = ka.a;
  extern __shared__ double sm[];
  __shared__ WCand wc[kLuppThreads / 32];
  __shared__ double sred[kLuppThreads / 32];
  __shared__ WCand s_best[2];
  const int G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ctid = threadIdx.x - 32;  // compute-thread id (warps 1..7)
  constexpr int kComp = kCompWarps * 32;
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
  const int smax = a.cols_max;
  const int stride = ka.pub_stride;
  double* Ws = sm;                                       // [smax][Rb]
  double* prow = Ws + static_cast<size_t>(smax) * Rb;    // [2][smax] pivot rows (by step parity)
  double* wtail = prow + 2 * smax;                       // [kLuppThreads/32][smax] warp winner tails
  double* F = wtail + (kLuppThreads / 32) * smax;        // [Rb] factors of the current step
  uint8_t* banned = reinterpret_cast<uint8_t*>(F + Rb);  // [Rb]

#pragma unroll 4
  for (int t = 0; t < steps; ++t)
    for (int r = threadIdx.x; r < nr; r += kLuppThreads) Ws[t * Rb + r] = a.W[(r0 + r) + t * a.ldw];
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
    for (int t = 0; t < steps; ++t)
      for (int r = threadIdx.x; r < nr; r += kLuppThreads) {
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
  const uint32_t gen = a.d_gen_k ? (a.gen_base | (static_cast<uint32_t>(*a.d_gen_k & 0x1FFFFF) << 1) |
                                     static_cast<uint32_t>(a.gen_which))
                                  : ka.gen;
  const uint64_t gen_hi = static_cast<uint64_t>(gen) << 32;

  // compute warps: warp candidate on column `col` + that row's tail (columns > col) into
  // wtail[warp]; `upd` = (factor lane value, pivot row) when the tail is an update
  auto warp_candidate = [&](WCand mine, int col, bool upd, const double* P) {
    const WCand w = warp_argmax(mine);
    if (w.key) {
      const int lr = w.idx - static_cast<int>(r0);
      const double f = upd ? F[lr] : 0.0;
      for (int t = col + 1 + lane; t < steps; t += 32)
        wtail[warp * smax + t] = upd ? __dsub_rn(Ws[t * Rb + lr], __dmul_rn(f, P[t])) : Ws[t * Rb + lr];
    }
    if (lane == 0) wc[warp] = w;
  };
  // warp 0: CTA candidate -> slot (parity of col), released with tag (gen, col + 1)
  auto publish = [&](int col) {
    const WCand c = (lane >= 1 && lane <= kCompWarps) ? wc[lane] : WCand{0ull, -1, -1.0};
    const WCand bc = warp_argmax(c);
    double* slot = ka.pub + (static_cast<size_t>(col & 1) * G + blockIdx.x) * stride;
    if (lane == 0) {
      slot[1] = key_mag(bc.key);
      slot[2] = bc.second;
      slot[3] = __longlong_as_double(bc.key ? static_cast<long long>(bc.idx) : -1ll);
    }
    if (bc.key) {
      const int lr = bc.idx - static_cast<int>(r0);
      const int ow = 1 + (lr % kComp) / 32;  // owning compute warp
      if (lane == 0) slot[4 + col] = Ws[col * Rb + lr];
      for (int t = col + 1 + lane; t < steps; t += 32) slot[4 + t] = wtail[ow * smax + t];
    }
    // __syncwarp orders the lanes' slot writes before lane 0's release store (cumulative)
    __syncwarp();
    if (lane == 0) st_release_u64(reinterpret_cast<uint64_t*>(slot), gen_hi | static_cast<uint64_t>(col + 1));
  };
  // warp 0: wait for every CTA's slot of step s, reduce, fetch the winner row
  auto exchange = [&](int s) {
    const double* pubs = ka.pub + static_cast<size_t>(s & 1) * G * stride;
    const uint64_t want = gen_hi | static_cast<uint64_t>(s + 1);
    WCand c{0ull, -1, -1.0};
    for (int q = lane; q < G; q += 32) {  // ascending q = ascending row slabs
      const double* slot = pubs + static_cast<size_t>(q) * stride;
      while (ld_acquire_u64(reinterpret_cast<const uint64_t*>(slot)) != want) {
      }
      const double mag = slot[1];
      if (mag >= 0.0) {
        const uint64_t k = mag_key(mag);
        if (k > c.key) {
          c.second = fmax(key_mag(c.key), slot[2]);
          c.key = k;
          c.idx = static_cast<int32_t>(__double_as_longlong(slot[3]));
        } else {
          c.second = fmax(c.second, mag);
        }
      }
    }
    const WCand best = warp_argmax(c);
    if (best.key) {
      const double* ws_ = pubs + static_cast<size_t>(best.idx / Rb) * stride;
      for (int t = s + lane; t < steps; t += 32) prow[(s & 1) * smax + t] = ws_[4 + t];
    }
    if (lane == 0) s_best[s & 1] = best;
  };

  // ---- step 0: candidates on column 0 ----
  if (warp > 0) {
    WCand mine{0ull, -1, -1.0};
    for (int r = ctid; r < nr; r += kComp)
      if (!banned[r]) mine = wcand_merge_row(mine, fabs(Ws[r]), static_cast<int32_t>(r0 + r));
    warp_candidate(mine, 0, false, nullptr);
  }
  __syncthreads();  // B2
  if (warp == 0) {
    publish(0);
    exchange(0);
  }
  __syncthreads();  // B1

  int count = 0;
  double first = 0.0;
  for (int s = 0; s < steps; ++s) {
    const WCand best = s_best[s & 1];
    const double best_mag = key_mag(best.key);
    if (best.key == 0 || best_mag <= abs_floor) break;
    if (s == 0)
      first = best_mag;
    else if (best_mag < a.pivot_floor * first)
      break;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.d_idx[s] = best.idx;
      a.d_best[s] = best_mag;
      a.d_second[s] = best.second;
    }
    ++count;
    if (s + 1 >= steps) break;
    const double* P = prow + (s & 1) * smax;
    if (warp > 0) {
      // column s+1 first (critical path), factors kept for the deferred columns
      const double pivot = P[s];
      WCand mine{0ull, -1, -1.0};
      for (int rr = ctid; rr < nr; rr += kComp) {
        if (banned[rr]) continue;
        if (r0 + rr == best.idx) {
          banned[rr] = 1;  // only the owning thread ever reads this flag
          continue;
        }
        const double f = __ddiv_rn(Ws[s * Rb + rr], pivot);
        F[rr] = f;
        const double v = __dsub_rn(Ws[(s + 1) * Rb + rr], __dmul_rn(f, P[s + 1]));
        Ws[(s + 1) * Rb + rr] = v;
        mine = wcand_merge_row(mine, fabs(v), static_cast<int32_t>(r0 + rr));
      }
      __syncwarp();
      warp_candidate(mine, s + 1, true, P);
    }
    __syncthreads();  // B2
    if (warp == 0) {
      publish(s + 1);
      exchange(s + 1);
    } else {
      // deferred columns s+2.. (overlaps the exchange)
      for (int rr = ctid; rr < nr; rr += kComp) {
        if (banned[rr]) continue;
        const double f = F[rr];
        for (int t0 = s + 2; t0 < steps; t0 += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = (t0 + u < steps) ? Ws[(t0 + u) * Rb + rr] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (t0 + u < steps) Ws[(t0 + u) * Rb + rr] = __dsub_rn(v[u], __dmul_rn(f, P[t0 + u]));
        }
      }
    }
    __syncthreads();  // B1
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
  }
}

// ---------------------------------------------------------------------------------
// Thread-block-cluster variant for small problems (W fits in the shared memory of one
// cluster of up to 16 CTAs): the per-step exchange goes through distributed shared memory
// and a cluster barrier instead of global memory and a grid-wide barrier. Each CTA keeps a
// contiguous slab of rows; per step it publishes (|best|, runner-up, index, row tail) in
// its own shared memory (double-buffered by step parity), all CTAs read the CL slots over
// DSMEM after the cluster barrier and reduce them in the same fixed order. Identical
// arithmetic to the kernels above.
// ---------------------------------------------------------------------------------
constexpr int kClusterThreads = 512;
constexpr int kClusterComp = kClusterThreads - 32;

struct LuppClusterArgs {
  LuppArgs a;
  long long* dbg;   // optional per-step clock64() trace of CTA 0 (benchmarking)
  int rows_per_cta;
  int slot_stride;  // doubles per published slot: 4 + steps_max (tag, mag, second, idx, tail)
};

// st.async: store 16 bytes into another CTA's shared memory and signal that CTA's mbarrier
// with the byte count (complete_tx); the receiver waits on its own barrier only.
__device__ __forceinline__ void st_async_v2(uint32_t remote_addr, double a, double b, uint32_t remote_mbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(remote_addr),
               "d"(a), "d"(b), "r"(remote_mbar)
               : "memory");
}
__device__ __forceinline__ uint32_t map_cluster_addr(uint32_t local_addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}

__device__ __forceinline__ void st_release_cluster_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.cluster.shared::cta.u64 [%0], %1;\n" ::"r"(smem_u32(p)), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_cluster_u64(const uint64_t* generic_remote) {
  uint64_t v;
  asm volatile("ld.acquire.cluster.u64 %0, [%1];\n" : "=l"(v) : "l"(generic_remote) : "memory");
  return v;
}

// Same pipelined schedule as lupp_smem_kernel, but the slots live in the publishing CTA's
// own shared memory and are read over distributed shared memory: the per-step exchange is
// a few DSMEM round trips inside one thread-block cluster (<= 16 CTAs) instead of L2 round
// trips across the whole GPU. Used whenever W fits in the cluster's shared memory.
__global__ void __launch_bounds__(kClusterThreads, 1) lupp_cluster_kernel(LuppClusterArgs ka) {
  cg::cluster_group cluster = cg::this_cluster();
  const LuppArgs& a = ka.a;
  extern __shared__ double sm[];
  __shared__ WCand wc[kClusterThreads / 32];
  __shared__ double sred[kClusterThreads / 32];
  __shared__ double s_norm;
  __shared__ WCand s_best[2];
  constexpr int kWarps = kClusterThreads / 32;
  const int CL = static_cast<int>(cluster.num_blocks());
  const int me = static_cast<int>(cluster.block_rank());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ctid = threadIdx.x - 32;
  const int Rb = ka.rows_per_cta;
  const int64_t r0 = static_cast<int64_t>(me) * Rb;
  int64_t nr64 = a.rows - r0;
  nr64 = nr64 < 0 ? 0 : (nr64 > Rb ? Rb : nr64);
  const int nr = static_cast<int>(nr64);
  int steps = a.cols_max;
  if (a.d_steps) steps = min(steps, *a.d_steps);
  if (steps <= 0) {
    if (me == 0 && threadIdx.x == 0) {
      *a.d_count = 0;
      if (a.d_width_out) *a.d_width_out = 0;
    }
    return;  // uniform across the cluster: no DSMEM traffic happened
  }
  const int smax = a.cols_max;
  const int stride = ka.slot_stride;
  double* Ws = sm;                                       // [smax][Rb]
  double* prow = Ws + static_cast<size_t>(smax) * Rb;    // [2][smax]
  double* wtail = prow + 2 * smax;                       // [kWarps][smax]
  double* F = wtail + kWarps * smax;                     // [Rb]
  // [2][CL][stride] every CTA's pushed slot (16-byte aligned: st.async writes pairs)
  double* inbox = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(F + Rb) + 15) & ~uintptr_t(15));
  double* stage = inbox + 2 * CL * stride;               // [stride] this CTA's outgoing slot
  uint8_t* banned = reinterpret_cast<uint8_t*>(stage + stride);  // [Rb]
  __shared__ __align__(8) uint64_t mbar[2];

  for (int t = 0; t < steps; ++t)
    for (int r = threadIdx.x; r < nr; r += kClusterThreads) Ws[t * Rb + r] = a.W[(r0 + r) + t * a.ldw];
  for (int r = threadIdx.x; r < nr; r += kClusterThreads) {
    const uint8_t mk = a.mask[r0 + r];
    banned[r] = (mk == 1 || mk == a.epoch) ? 1 : 0;
  }
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();

  double nsq;
  if (a.d_norm_sq) {
    nsq = *a.d_norm_sq;
    cluster.sync();  // every CTA's mbarriers are initialised before anyone pushes to them
  } else {
    double sq = 0.0;
    for (int t = 0; t < steps; ++t)
      for (int r = threadIdx.x; r < nr; r += kClusterThreads) {
        const double v = Ws[t * Rb + r];
        sq = fma(v, v, sq);
      }
    const double b = block_sum<kClusterThreads>(sq, sred);
    if (threadIdx.x == 0) s_norm = b;
    cluster.sync();
    nsq = 0.0;
    for (int q = 0; q < CL; ++q) nsq += *cluster.map_shared_rank(&s_norm, q);
  }
  const double abs_floor = 1e2 * 2.220446049250313e-16 * sqrt(nsq);

  auto warp_candidate = [&](WCand mine, int col, bool upd, const double* P) {
    const WCand w = warp_argmax(mine);
    if (w.key) {
      const int lr = w.idx - static_cast<int>(r0);
      const double f = upd ? F[lr] : 0.0;
      for (int t = col + 1 + lane; t < steps; t += 32)
        wtail[warp * smax + t] = upd ? __dsub_rn(Ws[t * Rb + lr], __dmul_rn(f, P[t])) : Ws[t * Rb + lr];
    }
    if (lane == 0) wc[warp] = w;
  };
  // warp 0: CTA candidate (mag, second, idx, row tail from `col`) pushed with st.async into
  // slot `me` of every CTA's inbox (parity of col); each receiver's mbarrier counts the bytes
  const uint32_t slot_bytes = static_cast<uint32_t>(stride) * 8u;
  auto publish = [&](int col) {
    const WCand c = (lane >= 1 && lane < kWarps) ? wc[lane] : WCand{0ull, -1, -1.0};
    const WCand bc = warp_argmax(c);
    const int par = col & 1;
    if (lane == 0) {
      stage[0] = key_mag(bc.key);
      stage[1] = bc.second;
      stage[2] = __longlong_as_double(bc.key ? static_cast<long long>(bc.idx) : -1ll);
      stage[3] = 0.0;
    }
    if (bc.key) {
      const int lr = bc.idx - static_cast<int>(r0);
      const int ow = 1 + (lr % kClusterComp) / 32;
      if (lane == 0) stage[4 + col] = Ws[col * Rb + lr];
      for (int t = col + 1 + lane; t < steps; t += 32) stage[4 + t] = wtail[ow * smax + t];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive_expect_tx(&mbar[par], static_cast<uint32_t>(CL) * slot_bytes);
    const uint32_t local_slot = smem_u32(inbox + (static_cast<size_t>(par) * CL + me) * stride);
    const uint32_t local_bar = smem_u32(&mbar[par]);
    const int pairs = stride / 2;
    for (int e = lane; e < CL * pairs; e += 32) {
      const int dst = e / pairs, pr = e - dst * pairs;
      const int t0 = 2 * pr;
      // columns < col of the tail are never read: send zeros instead of stale values
      const double v0 = (t0 < 4 || t0 - 4 >= col) ? stage[t0] : 0.0;
      const double v1 = (t0 + 1 < 4 || t0 - 3 >= col) ? stage[t0 + 1] : 0.0;
      st_async_v2(map_cluster_addr(local_slot + t0 * 8, dst), v0, v1, map_cluster_addr(local_bar, dst));
    }
  };
  // warp 0: wait for the CL pushed slots of step s, reduce them in fixed order, keep the
  // winner's row (all local reads)
  auto exchange = [&](int s) {
    const int par = s & 1;
    mbar_wait_cluster(&mbar[par], static_cast<uint32_t>((s >> 1) & 1));
    const double* box = inbox + static_cast<size_t>(par) * CL * stride;
    WCand c{0ull, -1, -1.0};
    if (lane < CL) {
      const double* rs = box + static_cast<size_t>(lane) * stride;
      const double mag = rs[0];
      if (mag >= 0.0) {
        c.key = mag_key(mag);
        c.idx = static_cast<int32_t>(__double_as_longlong(rs[2]));
        c.second = rs[1];
      }
    }
    const WCand best = warp_argmax(c);
    if (best.key) {
      const double* ws_ = box + static_cast<size_t>(best.idx / Rb) * stride;
      for (int t = s + lane; t < steps; t += 32) prow[par * smax + t] = ws_[4 + t];
    }
    if (lane == 0) s_best[par] = best;
  };

  if (warp > 0) {
    WCand mine{0ull, -1, -1.0};
    for (int r = ctid; r < nr; r += kClusterComp)
      if (!banned[r]) mine = wcand_merge_row(mine, fabs(Ws[r]), static_cast<int32_t>(r0 + r));
    warp_candidate(mine, 0, false, nullptr);
  }
  __syncthreads();
  if (warp == 0) {
    publish(0);
    exchange(0);
  }
  __syncthreads();

  int count = 0;
  double first = 0.0;
  long long* dbg = (ka.dbg && me == 0) ? ka.dbg : nullptr;
  double* lu_blk = a.lu_out ? a.lu_out + (a.d_lu_r ? *a.d_lu_r : 0) * a.lu_ld : nullptr;
  for (int s = 0; s < steps; ++s) {
    if (dbg && threadIdx.x == 32) dbg[s * 8 + 0] = clock64();
    const WCand best = s_best[s & 1];
    const double best_mag = key_mag(best.key);
    if (best.key == 0 || best_mag <= abs_floor) break;
    if (s == 0)
      first = best_mag;
    else if (best_mag < a.pivot_floor * first)
      break;
    if (me == 0 && threadIdx.x == 0) {
      a.d_idx[s] = best.idx;
      a.d_best[s] = best_mag;
      a.d_second[s] = best.second;
    }
    if (lu_blk && best.idx >= r0 && best.idx < r0 + nr) {
      // the pivot row is fully eliminated through step s-1: (multipliers, U(s, s:)) = LU row s
      const int lr = static_cast<int>(best.idx - r0);
      for (int t = threadIdx.x; t < steps; t += kClusterThreads) lu_blk[s + t * a.lu_ld] = Ws[t * Rb + lr];
    }
    ++count;
    if (s + 1 >= steps) break;
    const double* P = prow + (s & 1) * smax;
    if (warp > 0) {
      const double pivot = P[s];
      WCand mine{0ull, -1, -1.0};
      for (int rr = ctid; rr < nr; rr += kClusterComp) {
        if (banned[rr]) continue;
        if (r0 + rr == best.idx) {
          banned[rr] = 1;
          continue;
        }
        const double f = __ddiv_rn(Ws[s * Rb + rr], pivot);
        F[rr] = f;
        if (lu_blk) Ws[s * Rb + rr] = f;  // column s is dead for this row: keep its multiplier
        const double v = __dsub_rn(Ws[(s + 1) * Rb + rr], __dmul_rn(f, P[s + 1]));
        Ws[(s + 1) * Rb + rr] = v;
        mine = wcand_merge_row(mine, fabs(v), static_cast<int32_t>(r0 + rr));
      }
      __syncwarp();
      if (dbg && threadIdx.x == 32) dbg[s * 8 + 1] = clock64();
      warp_candidate(mine, s + 1, true, P);
      }
    __syncthreads();
    if (warp == 0) {
      if (dbg && threadIdx.x == 0) dbg[s * 8 + 3] = clock64();
      publish(s + 1);
      if (dbg && threadIdx.x == 0) dbg[s * 8 + 4] = clock64();
      exchange(s + 1);
      if (dbg && threadIdx.x == 0) dbg[s * 8 + 5] = clock64();
    } else {
      for (int rr = ctid; rr < nr; rr += kClusterComp) {
        if (banned[rr]) continue;
        const double f = F[rr];
        for (int t0 = s + 2; t0 < steps; t0 += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = (t0 + u < steps) ? Ws[(t0 + u) * Rb + rr] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (t0 + u < steps) Ws[(t0 + u) * Rb + rr] = __dsub_rn(v[u], __dmul_rn(f, P[t0 + u]));
        }
      }
      if (dbg && threadIdx.x == 32) dbg[s * 8 + 6] = clock64();
    }
    __syncthreads();
    if (dbg && threadIdx.x == 32) dbg[s * 8 + 7] = clock64();
  }
  if (me == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
  }
  cluster.sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
}


static long long* g_lupp_dbg = nullptr;
static long long* g_lupp_gdbg = nullptr;
static int g_force_path = 0;  // benchmarking: 0 automatic, 1 cluster, 2 grid smem, 3 global

// ---------------------------------------------------------------------------------
// Cluster LUPP, v2 (the default cluster path). Same pivots and arithmetic as above, with a
// much shorter per-step critical path:
//  * division by the pivot through its correctly rounded reciprocal and one FMA correction
//    (Markstein): q = RN(a*y), r = fma(-q, p, a), RN(q + r*y) equals RN(a/p) when
//    y = RN(1/p) and nothing under/overflows; outside a safe exponent window it falls back
//    to IEEE division (tools/microbench/div_check.cu: 7.6e10 pairs, 0 differences). The
//    reciprocal is formed once per step by the exchange warp, off the row loop;
//  * a thread's rows (at most RMAX) are handled together; their liveness is a register
//    bitmask, indices are 32-bit;
//  * after the CTA barrier every warp w < CL redundantly reduces the CTA's warp candidates
//    and pushes the CTA slot (|v|, runner-up, row, then the candidate's row tail) into CTA
//    w's inbox with st.async — 16 pushes in parallel instead of one warp doing all of them —
//    and the exchange warp reduces its own inbox (all reads local).
// The inbox is double-buffered by step parity; a CTA writes a parity again only after an
// exchange that needed every CTA's next push, which each CTA issues after it finished
// reading the earlier one.
// ---------------------------------------------------------------------------------
struct LuppClusterV2Args {
  LuppArgs a;
  long long* dbg;  // optional per-step clock64() trace of CTA 0 (16 slots per step)
  int skeleton;    // benchmarking only: 1 = skip the row eliminations (exchange cost alone)
  int serial_exchange;  // reduce the CL slots lane-serially instead of with warp collectives
  int rows_per_cta;
  int smax;        // column capacity of the buffers (cols_max)
  int slot;        // doubles per inbox slot: 4 + smax rounded up to even
};

// clock64() that issues only after `dep` is available (trace stamps after barriers / loads)
__device__ __forceinline__ long long clock_after(unsigned long long dep) {
  long long c;
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.u64 p, %1, 0x5a5a5a5a5a5a5a5a;\n@p mov.u64 %0, %%clock64;\n@!p mov.u64 %0, "
      "%%clock64;\n}\n"
      : "=l"(c)
      : "l"(dep)
      : "memory");
  return c;
}

// out-of-line IEEE division: the rare fallback stays out of the (instruction-cache
// sensitive) step loop
template <int THREADS, int RMAX>
__global__ void __launch_bounds__(THREADS, 1) lupp_cluster_v2_kernel(LuppClusterV2Args ka) {
  // warp roles: warps 0..3 (one per scheduler sub-partition) are service warps — each reduces
  // the CTA's warp candidates and pushes the CTA slot to a quarter of the cluster; warp 0 also
  // reduces the inbox — and warps 4.. own rows.
  constexpr int kWarps = THREADS / 32;
  constexpr int kSvc = 4;
  constexpr int kCompWarps = kWarps - kSvc;
  constexpr int kComp = kCompWarps * 32;
  constexpr int kPanel = 2;  // rank-1 updates of later columns are applied kPanel steps at a time
  cg::cluster_group cluster = cg::this_cluster();
  const LuppArgs& a = ka.a;
  extern __shared__ __align__(16) double sm[];
  __shared__ WCand wc[kCompWarps];
  __shared__ double sred[kWarps];
  __shared__ double s_norm;
  __shared__ WCand s_best[2];
  __shared__ double s_rcp[2];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ int64_t s_piv[64];  // this call's pivots (all CTAs know them): post gathers
  const int CL = static_cast<int>(cluster.num_blocks());
  const int me = static_cast<int>(cluster.block_rank());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool svc = warp < kSvc;
  const int cw = warp - kSvc;  // compute-warp index (valid when !svc)
  const int ctid = cw * 32 + lane;
  const int Rb = ka.rows_per_cta;
  const int smax = ka.smax, SL = ka.slot;
  const int r0 = me * Rb;
  const int nr = max(0, min(Rb, static_cast<int>(a.rows) - r0));
  griddep_wait();  // everything below reads the predecessor's output
  int steps = a.cols_max;
  if (a.begin_ctl) {
    // iteration begin (misc.cu iter_begin_kernel): every CTA derives the same step count from
    // the loop control; CTA 0 records it (the others never read what it writes)
    IterCtl* ctl = static_cast<IterCtl*>(a.begin_ctl);
    const int done = ctl->done;
    const bool budget_out = !done && (ctl->r >= ctl->max_rank || ctl->k >= ctl->max_iters);
    const int blk = (done || budget_out) ? 0 : static_cast<int>(min(static_cast<int64_t>(ctl->b), ctl->max_rank - ctl->r));
    steps = min(steps, blk);
    if (me == 0 && threadIdx.x == 0) {
      IterState* slot = static_cast<IterState*>(a.begin_slot);
      slot->ncols = slot->nrows = slot->width = 0;
      slot->valid = (done || budget_out) ? 0 : 1;
      if (budget_out) {
        ctl->done = 1;
        ctl->status = 1;  // MaxRank
      }
      if (!done) ctl->block = blk;
    }
  } else if (a.d_steps) {
    steps = min(steps, *a.d_steps);
  }
  if (steps <= 0) {
    if (me == 0 && threadIdx.x == 0) {
      *a.d_count = 0;
      if (a.d_width_out) *a.d_width_out = 0;
    }
    return;  // uniform across the cluster
  }
  double* Ws = sm;                                                     // [smax][Rb]
  double* U = Ws + static_cast<size_t>(smax) * Rb;                     // [smax][smax] pivot rows
  double* wtail = U + smax * smax;                                     // [kCompWarps][smax]
  double* inbox = reinterpret_cast<double*>(                           // [2][16][SL]
      (reinterpret_cast<uintptr_t>(wtail + kCompWarps * smax) + 15) & ~uintptr_t(15));

  uint32_t live = 0;  // bit k: row ctid + k*kComp is a candidate
  // slab load: every element an independent 8-byte cp.async, one wait for all of them
  for (int t = 0; t < steps; ++t)
    for (int r = threadIdx.x; r < nr; r += THREADS)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(Ws + t * Rb + r)),
                   "l"(a.W + (r0 + r) + t * a.ldw)
                   : "memory");
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  if (!svc) {
#pragma unroll
    for (int k = 0; k < RMAX; ++k) {
      const int rr = ctid + k * kComp;
      if (rr < nr) {
        const uint8_t mk = a.mask[r0 + rr];
        if (!(mk == 1 || mk == a.epoch)) live |= 1u << k;
      }
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_barrier_init();
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  double nsq;
  if (a.d_norm_sq) {
    nsq = *a.d_norm_sq;
    cluster.sync();  // every CTA's mbarriers are initialised before anyone pushes to them
  } else {
    double sq = 0.0;
    for (int t = 0; t < steps; ++t)
      for (int r = threadIdx.x; r < nr; r += THREADS) {
        const double v = Ws[t * Rb + r];
        sq = fma(v, v, sq);
      }
    const double b = block_sum<THREADS>(sq, sred);
    if (threadIdx.x == 0) s_norm = b;
    cluster.sync();
    nsq = 0.0;
    for (int q = 0; q < CL; ++q) nsq += *cluster.map_shared_rank(&s_norm, q);
  }
  const double abs_floor = 1e2 * 2.220446049250313e-16 * sqrt(nsq);
  double* lu_blk = a.lu_out ? a.lu_out + (a.d_lu_r ? *a.d_lu_r : 0) * a.lu_ld : nullptr;
#ifdef ITERCUR_LUPP_INSTRUMENT  // tracing / ablation build (tools/lupp_one.py with ITERCUR_LUPP_TRACE)
  long long* dbg = (ka.dbg && me == 0) ? ka.dbg : nullptr;
  const int kSkel = ka.skeleton, kSerial = ka.serial_exchange;
#else  // production: the instrumentation folds away
  long long* const dbg = nullptr;
  constexpr int kSkel = 0, kSerial = 0;
#endif

  // bytes one CTA pushes per step (header + pair-aligned tail from column col)
  auto push_pairs = [&](int col) { return 2 + (steps - (col & ~1) + 1) / 2; };
  // service warp sv: CTA candidate -> slot `me` of the inboxes of CTAs sv, sv + kSvc, ..
  auto push = [&](int col) {
    const int par = col & 1;
    const WCand c = lane < kCompWarps ? wc[lane] : WCand{0ull, -1, -1.0};
    const long long k10 = dbg ? clock_after(c.key) : 0;
    const WCand bc = warp_argmax(c);
    const long long k11 = dbg ? clock_after(bc.key) : 0;
    if (dbg && threadIdx.x == 0 && col > 0) {
      dbg[(col - 1) * 16 + 10] = k10;
      dbg[(col - 1) * 16 + 11] = k11;
    }
    const int npairs = push_pairs(col);
    if (lane < npairs) {
      double v0 = 0.0, v1 = 0.0;
      if (lane == 0) {
        v0 = bc.key ? key_mag(bc.key) : -1.0;
        v1 = bc.second;
      } else if (lane == 1) {
        v0 = __longlong_as_double(bc.key ? static_cast<long long>(bc.idx) : -1ll);
      } else if (bc.key) {
        // the CTA winner's row from column col on: column col was eliminated through step
        // col-1 by its owner (stored), later columns still owe the open panel's steps
        // s0..col-1, applied here in step order with the multipliers kept in Ws
        const int lr = bc.idx - r0;
        const int t0 = (col & ~1) + 2 * (lane - 2);
        const int sp = col - 1, jp = sp >= 0 ? sp % kPanel : -1, s0 = sp - jp;
        double fm[kPanel];
#pragma unroll
        for (int j = 0; j < kPanel; ++j) fm[j] = j <= jp ? Ws[(s0 + j) * Rb + lr] : 0.0;
        auto tail_at = [&](int t) {
          if (t < col || t >= steps) return 0.0;
          double x = Ws[t * Rb + lr];
          if (t > col) {
#pragma unroll
            for (int j = 0; j < kPanel; ++j)
              if (j <= jp) x = __dsub_rn(x, __dmul_rn(fm[j], U[(s0 + j) * smax + t]));
          }
          return x;
        };
        v0 = tail_at(t0);
        v1 = tail_at(t0 + 1);
      }
      const int t0 = (col & ~1) + 2 * (lane - 2);
      const int off = lane < 2 ? 2 * lane : 4 + t0;
      const uint32_t slot = smem_u32(inbox + (par * 16 + me) * SL + off);
      const uint32_t bar = smem_u32(&mbar[par]);
      if (dbg && threadIdx.x == 0 && col > 0)
        dbg[(col - 1) * 16 + 12] = clock_after(__double_as_longlong(v0) ^ __double_as_longlong(v1));
      for (int dst = warp; dst < CL; dst += kSvc)
        st_async_v2(map_cluster_addr(slot, dst), v0, v1, map_cluster_addr(bar, dst));
    }
  };
  // named barrier 1: the service warps have read the CTA winner's row (push), so the row
  // warps may apply a panel's trailing update to Ws
  auto tail_read_arrive = [&]() { asm volatile("bar.arrive 1, %0;\n" ::"n"(THREADS) : "memory"); };
  auto tail_read_wait = [&]() { asm volatile("bar.sync 1, %0;\n" ::"n"(THREADS) : "memory"); };
  // warp 0: wait for the CL slots of column col, reduce them in fixed order, copy the
  // winner's tail, form the next reciprocal
  auto exchange = [&](int col) {
    const int par = col & 1;
    if (lane == 0) mbar_wait_cluster(&mbar[par], static_cast<uint32_t>((col >> 1) & 1));
    __syncwarp();  // one poller; the warp leaves the wait converged
    const long long k5 = dbg ? clock64() : 0;
    WCand g{0ull, -1, -1.0};
    if (lane < CL) {
      const double* rs = inbox + (par * 16 + lane) * SL;
      const double mag = rs[0];
      if (mag >= 0.0) {
        g.key = mag_key(mag);
        g.idx = static_cast<int32_t>(__double_as_longlong(rs[2]));
        g.second = rs[1];
      }
    }
    const long long k13 = dbg ? clock_after(g.key) : 0;
    WCand best;
    if (kSerial) {
      // every lane scans the CL slots itself (broadcast shared loads, no warp collectives):
      // slots in rank order, strict '>' = lowest index on ties (rank order is index order)
      best = WCand{0ull, -1, -1.0};
      for (int q = 0; q < CL; ++q) {
        const double* rs = inbox + (par * 16 + q) * SL;
        const double mag = rs[0];
        if (mag < 0.0) continue;
        const uint64_t key = mag_key(mag);
        if (key > best.key) {
          best.second = fmax(key_mag(best.key), rs[1]);
          best.key = key;
          best.idx = static_cast<int32_t>(__double_as_longlong(rs[2]));
        } else {
          best.second = fmax(best.second, mag);
        }
      }
    } else {
      best = warp_argmax(g);
    }
    const long long k14 = dbg ? clock_after(best.key) : 0;
    if (kSkel >= 2 && dbg && col == 5) {  // benchmarking: cost of 100 ALU ops / 100 argmaxes here
      uint64_t x = best.key;
      const long long q0 = clock_after(x);
      if (kSkel == 2) {
        for (int q = 0; q < 100; ++q) x = x * 0x9e3779b97f4a7c15ull + (x >> 7);
      } else {
        WCand gg = g;
        for (int q = 0; q < 100; ++q) {
          const WCand bb = warp_argmax(gg);
          gg.key ^= (bb.key & 1);
          x ^= bb.key;
        }
      }
      const long long q1 = clock_after(x);
      if (lane == 0) dbg[(col - 1) * 16 + 9] = (q1 - q0) * 100 + (x & 1);
    }
    if (dbg && lane == 0 && col > 0) {
      dbg[(col - 1) * 16 + 5] = k5;
      dbg[(col - 1) * 16 + 13] = k13;
      dbg[(col - 1) * 16 + 14] = k14;
    }
    if (best.key) {
      // the winning slot's lane is its CTA rank (no division by the runtime slab size)
      const unsigned own = __ballot_sync(0xffffffffu, lane < CL && g.key == best.key && g.idx == best.idx);
      const double* ws_ = inbox + (par * 16 + (__ffs(own) - 1)) * SL + 4;
      for (int t = col + lane; t < steps; t += 32) U[col * smax + t] = ws_[t];
      if (lane == 0) s_rcp[par] = __drcp_rn(ws_[col]);
    }
    if (lane == 0) s_best[par] = best;
    if (dbg && lane == 0 && col > 0) dbg[(col - 1) * 16 + 15] = clock_after(__double_as_longlong(U[col * smax + steps - 1]));
  };

  // step-0 candidates: column 0 as loaded
  double cur[RMAX];      // this row's value in column s, eliminated through step s-1
  double fp[RMAX][kPanel];  // multipliers of the current panel's steps
#pragma unroll
  for (int k = 0; k < RMAX; ++k) {
    cur[k] = 0.0;
#pragma unroll
    for (int j = 0; j < kPanel; ++j) fp[k][j] = 0.0;
  }
  if (!svc) {
    WCand mine{0ull, -1, -1.0};
#pragma unroll
    for (int k = 0; k < RMAX; ++k) {
      const int rr = ctid + k * kComp;
      if (live >> k & 1) {
        cur[k] = Ws[rr];
        mine = wcand_merge_row(mine, fabs(cur[k]), r0 + rr);
      }
    }
    const WCand w = warp_argmax(mine);
    if (lane == 0) wc[cw] = w;
  }
  __syncthreads();
  if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&mbar[0], static_cast<uint32_t>(CL * push_pairs(0) * 16));
  if (svc) push(0);
  if (warp == 0) exchange(0);
  __syncthreads();

  int count = 0;
  double first = 0.0;
  for (int s = 0; s < steps; ++s) {
    if (dbg && threadIdx.x == 32) dbg[s * 16 + 0] = clock64();
    const WCand best = s_best[s & 1];
    const double best_mag = key_mag(best.key);
    if (best.key == 0 || best_mag <= abs_floor) break;
    if (s == 0)
      first = best_mag;
    else if (best_mag < a.pivot_floor * first)
      break;
    ++count;
    const bool last = s + 1 >= steps;
    if (last) griddep_launch_dependents();
    const int jp = s % kPanel, s0 = s - jp;  // position in the current panel
    const double* P = U + s * smax;
    if (threadIdx.x == 0) s_piv[s] = best.idx;
    if (svc) {
      if (warp == 0) {
        // bookkeeping and the LU row of D_k (owner CTA) while the compute warps eliminate
        if (me == 0 && lane == 0) {
          a.d_idx[s] = best.idx;
          a.d_best[s] = best_mag;
          a.d_second[s] = best.second;
        }
        if (lu_blk && best.idx >= r0 && best.idx < r0 + nr) {
          const int lr = best.idx - r0;
          for (int t = lane; t < steps; t += 32) lu_blk[s + t * a.lu_ld] = t < s ? Ws[t * Rb + lr] : P[t];
        }
        if (!last && lane == 0)
          mbar_arrive_expect_tx(&mbar[(s + 1) & 1], static_cast<uint32_t>(CL * push_pairs(s + 1) * 16));
      }
    } else if (!last) {
      const double pivot = P[s];
      const double y = s_rcp[s & 1];
      const bool p_ok = fabs(pivot) > 0x1p-968 && fabs(pivot) < 0x1p968;
      // the pivot row leaves the candidate set
      const int pk = best.idx - r0 - ctid;
      if (pk >= 0 && pk % kComp == 0 && pk / kComp < RMAX) live &= ~(1u << (pk / kComp));
      double ucol[kPanel];  // U(s0 + j, s + 1): the panel's pivot-row entries in column s+1
#pragma unroll
      for (int j = 0; j < kPanel; ++j) ucol[j] = j <= jp ? U[(s0 + j) * smax + s + 1] : 0.0;
      WCand mine{0ull, -1, -1.0};
      if (kSkel) mine = wcand_merge_row(mine, 1.0 + 1e-3 * ((ctid * 7 + s * 13) % 97), r0 + ctid);
      const uint32_t act = kSkel ? 0u : live;
      // branch-free over this thread's rows so their latencies overlap: loads, quotient
      // (Markstein), panel updates, then the (rare) IEEE fix-up, stores and merge
      double wn[RMAX], fq[RMAX];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < RMAX; ++k) {
        const int rr = min(ctid + k * kComp, Rb - 1);
        wn[k] = Ws[(s + 1) * Rb + rr];
        const double x = cur[k];
        const double q0 = __dmul_rn(x, y);
        const double rm = __fma_rn(-q0, pivot, x);
        fq[k] = __fma_rn(rm, y, q0);
        const double aq = fabs(fq[k]), ax = fabs(x);
        bad |= (act >> k & 1) && !(p_ok && aq > 0x1p-968 && aq < 0x1p968 && ax > 0x1p-968 && ax < 0x1p968);
      }
      if (__any_sync(0xffffffffu, bad)) {
#pragma unroll
        for (int k = 0; k < RMAX; ++k)
          if (act >> k & 1) fq[k] = div_by_pivot(cur[k], pivot, y, p_ok);
      }
#pragma unroll
      for (int k = 0; k < RMAX; ++k) {
#pragma unroll
        for (int j = 0; j < kPanel; ++j)
          if (j == jp) fp[k][j] = fq[k];
        // column s+1: eliminated through the previous panel in shared memory; apply this
        // panel's steps s0..s in order (the same operation sequence as right-looking)
        double v = wn[k];
#pragma unroll
        for (int j = 0; j < kPanel; ++j)
          if (j <= jp) v = __dsub_rn(v, __dmul_rn(fp[k][j], ucol[j]));
        if (act >> k & 1) {
          const int rr = ctid + k * kComp;
          Ws[s * Rb + rr] = fq[k];  // column s is dead for this row: keep its multiplier
          Ws[(s + 1) * Rb + rr] = v;  // column s+1, eliminated through step s
          cur[k] = v;
          const uint64_t key = mag_key(fabs(v));
          const bool better = key > mine.key;
          mine.second = better ? key_mag(mine.key) : fmax(mine.second, fabs(v));
          mine.key = better ? key : mine.key;
          mine.idx = better ? r0 + rr : mine.idx;
        }
      }
      if (dbg && threadIdx.x == 32) dbg[s * 16 + 1] = clock64();
      const WCand w = warp_argmax(mine);
      if (lane == 0) wc[cw] = w;
      if (dbg && threadIdx.x == 32) dbg[s * 16 + 2] = clock64();
    }
    if (last) break;
    __syncthreads();
    if (dbg && threadIdx.x == 0) dbg[s * 16 + 3] = clock_after(wc[0].key);
    if (svc) {
      push(s + 1);
      if (jp == kPanel - 1) tail_read_arrive();
      if (dbg && threadIdx.x == 0) dbg[s * 16 + 4] = clock64();
      if (warp == 0) {
        exchange(s + 1);
        if (dbg && lane == 0) dbg[s * 16 + 6] = clock64();
      }
    } else if (jp == kPanel - 1) {
      tail_read_wait();  // the service warps have read the CTA winner's row
      // panel end: apply the panel's kPanel rank-1 updates to columns s+2.. in one pass
      // (each element read and written once per panel instead of once per step)
      const double* Up = U + s0 * smax;
#pragma unroll
      for (int k = 0; k < RMAX; ++k) {
        if (!(live >> k & 1)) continue;
        const int rr = ctid + k * kComp;
        for (int t = s + 2; t < steps; ++t) {
          double x = Ws[t * Rb + rr];
#pragma unroll
          for (int j = 0; j < kPanel; ++j) x = __dsub_rn(x, __dmul_rn(fp[k][j], Up[j * smax + t]));
          Ws[t * Rb + rr] = x;
        }
      }
      if (dbg && threadIdx.x == 32) dbg[s * 16 + 7] = clock64();
    }
    __syncthreads();
    if (dbg && threadIdx.x == 32) dbg[s * 16 + 8] = clock_after(s_best[(s + 1) & 1].key);
  }
  if (me == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
  }
  // post gathers indexed by the pivots (replacing separate gather launches), spread over the
  // cluster's threads
  __syncthreads();
#pragma unroll
  for (int gq = 0; gq < 2; ++gq) {
    const LuppArgs::Gather& G = a.post[gq];
    if (!G.src) continue;
    const int64_t K = G.k_cap ? min(G.kmax, *G.k_cap) : G.kmax;
    const int64_t total = K * G.w_fill;
    const int64_t stride = static_cast<int64_t>(CL) * THREADS;
    for (int64_t e = static_cast<int64_t>(me) * THREADS + threadIdx.x; e < total; e += stride) {
      const int64_t q = e / K, kk = e - q * K;
      G.out[kk + q * G.ldo] = q < count ? G.src[kk * G.row_stride + s_piv[q] * G.col_stride] : 0.0;
    }
  }
  cluster.sync();  // no CTA leaves while a peer may still push into it
}

static size_t v2_smem_bytes(int threads, int smax, int Rb, int slot) {
  const int comp_warps = threads / 32 - 4;
  return sizeof(double) * (static_cast<size_t>(smax) * Rb + static_cast<size_t>(smax) * smax + comp_warps * smax + 2 +
                           2 * 16 * static_cast<size_t>(slot)) +
         16;
}

template <int THREADS, int RMAX>
static cudaError_t launch_cluster_v2(const LuppClusterV2Args& ka, int cl, size_t smem, cudaStream_t st) {
  return launch_ex(lupp_cluster_v2_kernel<THREADS, RMAX>, dim3(cl), dim3(THREADS), smem, st, dim3(cl, 1, 1), ka);
}

template <int THREADS, int RMAX>
static bool prepare_cluster_v2(size_t budget) {
  auto k = lupp_cluster_v2_kernel<THREADS, RMAX>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(budget)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = budget;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, k, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return clusters >= 1;
}

struct V2Plan {
  bool ok = false;
  int cl = 0, threads = 0, Rb = 0, slot = 0;
  size_t smem = 0;
};
static V2Plan plan_lupp_cluster_v2(const LuppArgs& a);

static cudaError_t try_lupp_cluster_v2(const LuppArgs& a, cudaStream_t st, int* grid_used) {
  const V2Plan pl = plan_lupp_cluster_v2(a);
  if (!pl.ok) return cudaErrorNotSupported;
  LuppClusterV2Args ka;
  ka.a = a;
  ka.dbg = g_lupp_dbg;
  ka.skeleton = getenv("ITERCUR_LUPP_SKELETON") ? atoi(getenv("ITERCUR_LUPP_SKELETON")) : 0;
  ka.serial_exchange = env_flag("ITERCUR_LUPP_SERIAL");
  ka.rows_per_cta = pl.Rb;
  ka.smax = std::max(a.cols_max, 1);
  ka.slot = pl.slot;
  if (grid_used) *grid_used = -100 - pl.cl;
  if (pl.threads == 768)
    return pl.Rb <= 640 ? launch_cluster_v2<768, 1>(ka, pl.cl, pl.smem, st)   // one row per row thread
                        : launch_cluster_v2<768, 2>(ka, pl.cl, pl.smem, st);
  return launch_cluster_v2<512, 4>(ka, pl.cl, pl.smem, st);
}

bool lupp_fuses_iteration_work(const LuppArgs& a) {
  return (g_force_path == 0 || g_force_path == 1) && plan_lupp_cluster_v2(a).ok;
}

static V2Plan plan_lupp_cluster_v2(const LuppArgs& a) {
  V2Plan pl;
  const int smax = std::max(a.cols_max, 1);
  const size_t budget = 225 * 1024;
  static int ready = -1;  // bit 0: 512-thread kernel usable, bit 1: 768-thread kernel usable
  if (ready < 0)
    ready = (prepare_cluster_v2<512, 4>(budget) ? 1 : 0) |
            (prepare_cluster_v2<768, 2>(budget) && prepare_cluster_v2<768, 1>(budget) ? 2 : 0);
  static const bool disabled = env_flag("ITERCUR_LUPP_NO_CLUSTER");
  static const bool v1 = env_flag("ITERCUR_LUPP_CLUSTER_V1");  // A/B switch
  static const int force_threads = [] {
    const char* e = getenv("ITERCUR_LUPP_THREADS");
    return e ? atoi(e) : 0;
  }();
  if (disabled || v1 || !ready || a.rows >= (1ll << 31) - 1 || smax > 56) return pl;
  const int slot = static_cast<int>(round_up(4 + smax + 1, 2));
  for (int cl = 1; cl <= 16; cl *= 2) {
    const int Rb = static_cast<int>(ceil_div(a.rows, cl));
    // 768 threads (20 row warps, <= 2 rows each) when the slab allows, else 512 (12 row
    // warps, <= 4 rows each); ITERCUR_LUPP_THREADS=512|768 forces one for A/B runs
    const bool big = force_threads != 512 && (ready & 2) && Rb <= 2 * 640;
    const int threads = big ? 768 : 512;
    if (!big && (!(ready & 1) || Rb > 4 * 384)) continue;
    const size_t smem = v2_smem_bytes(threads, smax, Rb, slot);
    if (smem > budget) continue;
    if (cl < 16 && Rb > 512) continue;  // spread slabs over more SMs: fewer rows per thread per step
    pl.ok = true;
    pl.cl = cl;
    pl.threads = threads;
    pl.Rb = Rb;
    pl.slot = slot;
    pl.smem = smem;
    return pl;
  }
  return pl;
}


static int cluster_capacity_ok(int cl, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, lupp_cluster_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return clusters;
}

// Try the cluster path; returns cudaErrorNotSupported when the problem does not fit.
static cudaError_t try_lupp_cluster(const LuppArgs& a, cudaStream_t st, int* grid_used) {
  const int steps = std::max(a.cols_max, 1);
  static bool attr_done = false;
  static bool usable = false;
  static int max_cl = 16;
  const size_t budget = 220 * 1024;
  if (!attr_done) {
    attr_done = true;
    usable = cudaFuncSetAttribute(lupp_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                 cudaSuccess &&
             cudaFuncSetAttribute(lupp_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(budget)) == cudaSuccess;
    if (usable && cluster_capacity_ok(16, budget) < 1) max_cl = 8;
    if (usable && cluster_capacity_ok(max_cl, budget) < 1) usable = false;
    cudaGetLastError();
  }
  static const bool disabled = env_flag("ITERCUR_LUPP_NO_CLUSTER");  // tuning switch
  if (disabled || !usable || a.rows >= (1ll << 31) - 1) return cudaErrorNotSupported;
  // smallest cluster whose slabs fit
  for (int cl = 1; cl <= max_cl; cl *= 2) {
    const int Rb = static_cast<int>(ceil_div(a.rows, cl));
    const int stride = static_cast<int>(round_up(steps + 4, 2));
    const size_t smem = sizeof(double) * (static_cast<size_t>(steps) * Rb + (2 + kClusterThreads / 32) * steps +
                                          Rb + 2 + (2 * cl + 1) * stride) + Rb + 16;
    if (smem > budget) continue;
    // enough rows per CTA to keep 1024 threads busy; prefer more CTAs for big slabs
    if (cl < max_cl && Rb > 2 * kClusterComp) continue;  // keep every compute thread to <= 2 rows
    LuppClusterArgs ka;
    ka.a = a;
    ka.dbg = g_lupp_dbg;
    ka.rows_per_cta = Rb;
    ka.slot_stride = stride;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (grid_used) *grid_used = -cl;
    return cudaLaunchKernelEx(&cfg, lupp_cluster_kernel, ka);
  }
  return cudaErrorNotSupported;
}

// ---------------------------------------------------------------------------------
// Grid-wide LUPP with panel-blocked updates, for slabs too large for shared memory (configs
// 4/5: 100000-200000 rows). The right-looking kernel above rewrites every remaining column
// of every row per pivot step — HBM-bound at these sizes. Here a thread keeps its rows'
// current column and the open panel's multipliers in registers: per step it reads one column
// and writes its multiplier; the later columns receive the panel's kPanelG rank-1 updates in
// one pass at the panel end (each element read and written once per panel). The pivot row
// for step s is rebuilt by every CTA from the winner's row in W (current through the last
// panel end), its stored multipliers and the panel's previous pivot rows (same operations in
// the same order as right-looking, so identical pivots). In-call bans live in registers;
// the pivot rows' LU factors are emitted for the row selection (no separate factorisation).
// ---------------------------------------------------------------------------------
// Panel-kernel candidate exchange. Merge of one candidate into a running one with the
// reference's rule (larger |value|, ties -> lower row index; the loser's magnitude feeds the
// runner-up).
__device__ __forceinline__ void wcand_merge(WCand& c, uint64_t key, int32_t idx, double second) {
  if (key > c.key || (key == c.key && key != 0 && idx < c.idx)) {
    c.second = fmax(second, key_mag(c.key));
    c.key = key;
    c.idx = idx;
  } else {
    c.second = fmax(c.second, key_mag(key));
  }
}
// Every warp reduces all G CTA candidates (lane-strided loads, then redux.sync).
__device__ __forceinline__ Cand panel_reduce_list(const Cand* cs, int G) {
  WCand c{0ull, 0x7fffffff, -1.0};
  constexpr int B = 8;  // loads of a batch issued together (one L2 round trip per batch)
  for (int q0 = threadIdx.x & 31; q0 < G; q0 += 32 * B) {
    Cand x[B];
#pragma unroll
    for (int u = 0; u < B; ++u) x[u] = q0 + 32 * u < G ? cs[q0 + 32 * u] : cand_empty();
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (x[u].idx >= 0) wcand_merge(c, mag_key(x[u].mag), static_cast<int32_t>(x[u].idx), x[u].second);
  }
  const WCand w = warp_argmax(c);
  return w.key ? Cand{key_mag(w.key), w.second, static_cast<int64_t>(w.idx)} : cand_empty();
}
// This CTA's candidate to global: warp argmax, then thread 0 merges the warps. With `arrivals`,
// thread 0 then announces it with a gpu-scope release increment (the CTA barrier before orders
// every thread's W stores of this step before it): the next step's readers wait on the count
// instead of a grid barrier.
__device__ __forceinline__ void panel_publish(const Cand& local, WCand* sw, Cand* out,
                                              unsigned long long* arrivals = nullptr) {
  WCand c{0ull, 0x7fffffff, -1.0};
  if (local.idx >= 0) wcand_merge(c, mag_key(local.mag), static_cast<int32_t>(local.idx), local.second);
  const WCand w = warp_argmax(c);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    WCand r = sw[0];
    for (int q = 1; q < kLuppThreads / 32; ++q)
      if (sw[q].key) wcand_merge(r, sw[q].key, sw[q].idx, sw[q].second);
    *out = r.key ? Cand{key_mag(r.key), r.second, static_cast<int64_t>(r.idx)} : cand_empty();
    if (arrivals) asm volatile("red.release.gpu.global.add.u64 [%0], 1;\n" ::"l"(arrivals) : "memory");
  }
}
// Wait until `target` CTA candidates have been announced: one poller per CTA (acquire at gpu
// scope, as cooperative groups' grid barrier polls), then the CTA barrier.
__device__ __forceinline__ void panel_wait(const unsigned long long* arrivals, unsigned long long target) {
  if (threadIdx.x == 0) {
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(arrivals) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// PG: panel width (8; 4 for the 8-rows-per-thread variant, whose multipliers must still fit
// in registers at 512 threads per CTA)
template <int RMAX, int PG>
__global__ void __launch_bounds__(kLuppThreads, 2) lupp_panel_kernel(LuppKernelArgs ka) {
  cg::grid_group grid = cg::this_grid();
  const LuppArgs& a = ka.a;
  extern __shared__ double sm[];  // P [smax] + U [PG][smax] + F [PG][RMAX][threads]
  __shared__ Cand sc[kLuppThreads / 32 + 1];
  __shared__ double sred[kLuppThreads / 32];
  __shared__ WCand sw[kLuppThreads / 32];
  const int smax = a.cols_max;
  double* P = sm;
  double* U = sm + smax;
  double* F = U + PG * smax;  // this thread's panel multipliers: F[(j * RMAX + k) * threads + tid]
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * kLuppThreads + threadIdx.x;
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * kLuppThreads;
  const int G = gridDim.x;
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
  double nsq;
  if (a.d_norm_sq) {
    nsq = *a.d_norm_sq;
  } else {
    double sq = 0.0;
    for (int t = 0; t < steps; ++t)
      for (int64_t i = gtid; i < a.rows; i += gstride) {
        const double v = W[i + t * ldw];
        sq = fma(v, v, sq);
      }
    const double b = block_sum<kLuppThreads>(sq, sred);
    if (threadIdx.x == 0) ka.norm_part[blockIdx.x] = b;
    grid.sync();
    nsq = 0.0;
    for (int q = 0; q < G; ++q) nsq += ka.norm_part[q];
  }
  const double abs_floor = 1e2 * 2.220446049250313e-16 * sqrt(nsq);
  double* lu_blk = a.lu_out ? a.lu_out + (a.d_lu_r ? *a.d_lu_r : 0) * a.lu_ld : nullptr;

  // this thread's rows i = gtid + k*gstride; live bits; current column; panel multipliers
  uint32_t live = 0;
  double cur[RMAX], nxt[RMAX];  // nxt: W(i, s+1) through the last panel end (prefetched)
  Cand local = cand_empty();
#pragma unroll
  for (int k = 0; k < RMAX; ++k) {
    const int64_t i = gtid + k * gstride;
    cur[k] = 0.0;
    nxt[k] = 0.0;
    if (i < a.rows) {
      const uint8_t mk = a.mask[i];
      if (!(mk == 1 || mk == a.epoch)) {
        live |= 1u << k;
        cur[k] = W[i];
        if (steps > 1) nxt[k] = W[i + ldw];
        local = cand_merge(local, Cand{fabs(cur[k]), -1.0, i});
      }
    }
  }
  Cand bc = block_reduce_cand(local, sc);
  if (threadIdx.x == 0) ka.cand[blockIdx.x] = bc;
  // the arrival count before any CTA of this launch increments it (increments start after this
  // barrier): step s waits for base + s * G announcements
  unsigned long long base = 0;
  if (ka.arrivals) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(base) : "l"(ka.arrivals) : "memory");
  grid.sync();

  int count = 0;
  double first = 0.0;
  long long* const dbg = (ka.dbg && blockIdx.x == 0 && threadIdx.x == 0) ? ka.dbg : nullptr;
  for (int s = 0; s < steps; ++s) {
    Cand best;
    if (ka.arrivals) {
      // one warp per CTA reads and reduces the CTA-candidate list (every warp reading it put eight
      // times the requests on the few L2 lines that hold it), then hands the winner to the others
      if (s > 0) panel_wait(ka.arrivals, base + static_cast<unsigned long long>(s) * G);
      if (dbg) dbg[s * 8 + 0] = clock64();
      if (threadIdx.x < 32) {
        const Cand c = panel_reduce_list(ka.cand + (s & 1) * G, G);
        if (threadIdx.x == 0) sc[kLuppThreads / 32] = c;
      }
      __syncthreads();
      best = sc[kLuppThreads / 32];
    } else {
      if (dbg) dbg[s * 8 + 0] = clock64();
      // every warp reduces the whole CTA-candidate list itself: no block barrier on this path
      best = panel_reduce_list(ka.cand + (s & 1) * G, G);
    }
    if (best.idx < 0 || best.mag <= abs_floor) break;
    if (s == 0)
      first = best.mag;
    else if (best.mag < a.pivot_floor * first)
      break;
    if (dbg) dbg[s * 8 + 1] = clock64();
    const int jp = s % PG, s0 = s - jp;
    // pivot row: the winner's row through the last panel end, then this panel's steps (all the
    // loads of the winner's row — values and panel multipliers — in one round trip)
    if (s + threadIdx.x < steps) {
      double mult[PG - 1];
#pragma unroll
      for (int j = 0; j < PG - 1; ++j) mult[j] = j < jp ? W[best.idx + (s0 + j) * ldw] : 0.0;
      for (int t = s + threadIdx.x; t < steps; t += kLuppThreads) {
        double x = W[best.idx + t * ldw];
#pragma unroll
        for (int j = 0; j < PG - 1; ++j)
          if (j < jp) x = __dsub_rn(x, __dmul_rn(mult[j], U[j * smax + t]));
        P[t] = x;
        U[jp * smax + t] = x;
      }
    }
    __syncthreads();
    if (dbg) dbg[s * 8 + 2] = clock64();
    if (blockIdx.x == 0) {
      if (threadIdx.x == 0) {
        a.d_idx[s] = best.idx;
        a.d_best[s] = best.mag;
        a.d_second[s] = best.second;
      }
      if (lu_blk)  // LU row s of D_k: multipliers (stored in W) then U(s, s:)
        for (int t = threadIdx.x; t < steps; t += kLuppThreads)
          lu_blk[s + t * a.lu_ld] = t < s ? W[best.idx + t * ldw] : P[t];
    }
    ++count;
    if (s + 1 >= steps) break;
    const double pivot = P[s], y = __drcp_rn(pivot);
    const bool p_ok = fabs(pivot) > 0x1p-968 && fabs(pivot) < 0x1p968;
    // (the panel must close exactly every PG steps: the pivot rows are rebuilt with the
    // open panel's terms, so a column may never receive them from a trailing update as well)
    const bool panel_end = jp == PG - 1;
    local = cand_empty();
#pragma unroll
    for (int k = 0; k < RMAX; ++k) {
      if (!(live >> k & 1)) continue;
      const int64_t i = gtid + k * gstride;
      if (i == best.idx) {
        live &= ~(1u << k);
        continue;
      }
      const double f = div_by_pivot(cur[k], pivot, y, p_ok);
      F[(jp * RMAX + k) * kLuppThreads + threadIdx.x] = f;
      W[i + s * ldw] = f;  // column s is dead for this row: its multiplier (LU factors, pivot rows)
      double v = nxt[k];
      for (int j = 0; j < jp; ++j)
        v = __dsub_rn(v, __dmul_rn(F[(j * RMAX + k) * kLuppThreads + threadIdx.x], U[j * smax + s + 1]));
      v = __dsub_rn(v, __dmul_rn(f, U[jp * smax + s + 1]));
      cur[k] = v;
      if (!panel_end && s + 2 < steps) nxt[k] = W[i + (s + 2) * ldw];  // raw next column, in flight across the barrier
      local = cand_merge(local, Cand{fabs(v), -1.0, i});
    }
    if (dbg) dbg[s * 8 + 3] = clock64();
    if (panel_end) {
      // close the panel: columns s+1.. of this thread's rows receive the panel's updates in one
      // pass, a chunk of C columns loaded together (latency bound otherwise)
#pragma unroll
      for (int k = 0; k < RMAX; ++k) {
        if (!(live >> k & 1)) continue;
        const int64_t i = gtid + k * gstride;
        double fr[PG];
#pragma unroll
        for (int j = 0; j < PG; ++j) fr[j] = F[(j * RMAX + k) * kLuppThreads + threadIdx.x];
        W[i + (s + 1) * ldw] = cur[k];
        constexpr int C = 8;
        for (int t0 = s + 2; t0 < steps; t0 += C) {
          double x[C];
#pragma unroll
          for (int u = 0; u < C; ++u) x[u] = t0 + u < steps ? W[i + (t0 + u) * ldw] : 0.0;
#pragma unroll
          for (int u = 0; u < C; ++u) {
            const int t = min(t0 + u, steps - 1);
#pragma unroll
            for (int j = 0; j < PG; ++j) x[u] = __dsub_rn(x[u], __dmul_rn(fr[j], U[j * smax + t]));
            if (t0 + u < steps) W[i + (t0 + u) * ldw] = x[u];
          }
          if (t0 == s + 2) nxt[k] = x[0];
        }
      }
    }
    if (dbg) dbg[s * 8 + 4] = clock64();
    panel_publish(local, sw, ka.cand + ((s + 1) & 1) * G + blockIdx.x, ka.arrivals);
    if (dbg) dbg[s * 8 + 5] = clock64();
    if (!ka.arrivals) grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
  }
}

// ---------------------------------------------------------------------------------
// Resident grid LUPP (round 2): the whole slab stays on chip for the call — one CTA per SM owns
// a contiguous block of at most 704 rows, one row per thread, the row's last KR columns in that
// thread's registers and its leading columns in shared memory (config 4: 100000 x 50 = 40 MB
// over 148 SMs' registers + shared memory). Per pivot step the slab is never re-read from L2;
// the only global traffic is the candidate exchange, and that exchange needs no fence, atomic
// or barrier: every (step, CTA) has its own record (header + the candidate row's tail) in a
// region cleared to an all-ones sentinel before the call (by the previous call, which clears
// the other of two regions), each word is written exactly once, so a reader that sees a word
// different from the sentinel sees its final value. One warp per CTA polls the step's headers,
// reduces them in the reference's order, then polls the winner's tail (two L2 round trips).
//   step s: [B1] f = W(i,s)/pivot (Markstein), column s+1 updated first, warp argmax; [B2] the
//   CTA winner's owner publishes its tail (columns > s+1 updated on the fly) while every row
//   applies the rest of the step's update — overlapped with the exchange of step s+1.
// Same per-element arithmetic as the kernels above (separate multiply and subtract roundings,
// correctly rounded division), so the pivot sequence is the reference's bit for bit. The pivot
// rows' LU factors (row s of D_k = multipliers of steps < s, then the pivot row) are written
// by the thread that owns the pivot row.
// ---------------------------------------------------------------------------------
constexpr int kResThreads = 384;  // warp 0: exchange; warps 1..11: two rows per thread
constexpr int kResWarps = kResThreads / 32;
constexpr int kResRowThreads = kResThreads - 32;
constexpr int kResRPT = 2;  // rows per row thread: local rows lr and lr + kResRowThreads
constexpr int kResKR = 16;  // trailing columns per row held in registers
constexpr int kResMaxSteps = 64;
constexpr int kResPanel = 4;              // shared-memory columns updated once per 4 pivot steps
constexpr int kResRing = 8;  // pivot rows kept (>= kResPanel + 1; a power of two: slot = step & 7)
constexpr int kResMaxG = 148;
constexpr int kResRec = 4 + kResMaxSteps;  // words 0-1 unused, 2 runner-up key, 3 unused, 4 + t the row
// region: norm partials [kResMaxG], compact headers [step][CTA][2] (a warp's poll touches 4 lines),
// records [step][CTA][kResRec] (word 2 runner-up key, 3 RN(1/pivot), 4 + t the row)
constexpr size_t kResHdrWords = static_cast<size_t>(kResMaxSteps) * kResMaxG * 2;
constexpr size_t kResRegionWords = kResMaxG + kResHdrWords + static_cast<size_t>(kResMaxSteps) * kResMaxG * kResRec;
constexpr uint64_t kResEmpty = ~0ull;
constexpr uint64_t kResMagic = 0x1C0B200A5A5E0002ull;
constexpr size_t kResScratchBytes = 64 + 2 * kResRegionWords * sizeof(uint64_t);

struct LuppResArgs {
  LuppArgs a;
  uint64_t* ctl;     // [0] magic, [1] call counter (region parity), [2] exchange time-out flag
  uint64_t* region;  // two regions of kResRegionWords: norm partials [kResMaxG], records [step][CTA]
  int rows_per_cta;
  long long* dbg;    // optional per-step clock64() trace of CTA 0 (8 slots per step)
  long long* gdbg;   // optional per-step globaltimer stamps of every CTA: [step][CTA][published, headers, tail]
  int backoff_ns;    // experiments: sleep between polls of an unpublished record
};

#if defined(ITERCUR_RES_LD_CG)
#define ITERCUR_RES_LD "ld.global.cg"
#elif defined(ITERCUR_RES_LD_VOLATILE)
#define ITERCUR_RES_LD "ld.volatile.global"
#else
#define ITERCUR_RES_LD "ld.relaxed.gpu.global"
#endif
__device__ __forceinline__ uint64_t res_ld(const uint64_t* p) {
  uint64_t v;
  asm volatile(ITERCUR_RES_LD ".u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void res_ld2(const uint64_t* p, uint64_t& x, uint64_t& y) {
  asm volatile(ITERCUR_RES_LD ".v2.u64 {%0, %1}, [%2];\n" : "=l"(x), "=l"(y) : "l"(p) : "memory");
}
__device__ __forceinline__ void res_st(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void res_st2(uint64_t* p, uint64_t x, uint64_t y) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n" ::"l"(p), "l"(x), "l"(y) : "memory");
}
// a row value as a record word: never the sentinel (a NaN with every bit set becomes the
// canonical quiet NaN; finite inputs never produce it)
__device__ __forceinline__ uint64_t res_enc(double v) {
  const uint64_t u = static_cast<uint64_t>(__double_as_longlong(v));
  return u == kResEmpty ? 0x7FF8000000000000ull : u;
}
__device__ __forceinline__ uint64_t res_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}
constexpr uint64_t kResTimeoutNs = 2000000000ull;  // a lost record ends the call instead of hanging

// Shared-memory column t of the resident LUPP is brought current at the steps s' = t (mod
// kResPanel) with s' <= t - 2; before the update pass of step s it is current through the last
// such s' <= s - 1 (-1: still the input). Its pending steps are (res_last_update(t, s), s].
__device__ __forceinline__ int res_last_update(int t, int s) {
  const int m = min(s - 1, t - 2);
  if (m < 0) return -1;
  int r = (m - t) % kResPanel;
  if (r < 0) r += kResPanel;
  return m - r < 0 ? -1 : m - r;
}

template <int KR>
__global__ void __launch_bounds__(kResThreads, 1) lupp_resident_kernel(LuppResArgs ka) {
  const LuppArgs& a = ka.a;
  extern __shared__ double Ws[];  // [R0][ldS]: columns 0..R0-1 of the CTA's rows (odd ldS: no bank conflicts along a row)
  __shared__ double Pr[kResRing][kResMaxSteps];  // pivot rows of the open panel + the next step
  __shared__ double stage[kResWarps][kResKR + 2];  // each row warp's winner: register columns, multiplier, next-column value
  __shared__ double emit[kResKR];  // the retired pivot row's register columns (its LU row)
  __shared__ WCand wc[kResWarps];
  __shared__ WCand s_best;
  __shared__ double s_y, s_nsq;
  __shared__ double s_red[kResWarps];
  __shared__ int s_abort;
  const int G = gridDim.x, g = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = threadIdx.x - 32;  // row threads: local rows lr and lr + kResRowThreads
  const int Rb = ka.rows_per_cta, ldS = Rb | 1;
  const int64_t r0 = static_cast<int64_t>(g) * Rb;
  int64_t nr64 = a.rows - r0;
  nr64 = nr64 < 0 ? 0 : (nr64 > Rb ? Rb : nr64);
  const int nr = static_cast<int>(nr64);
  int steps = a.cols_max;
  if (a.d_steps) steps = min(steps, *a.d_steps);
  if (steps <= 0) {
    if (g == 0 && threadIdx.x == 0) {
      *a.d_count = 0;
      if (a.d_width_out) *a.d_width_out = 0;
    }
    return;
  }
  const int R0 = steps > KR ? steps - KR : 0;  // columns [R0, steps) live in registers
  const int64_t ldw = a.ldw;

  // region of this call (parity of the call counter); the other region is cleared for the next
  // call. First use of a scratch buffer (no magic yet): clear this call's region too, grid-wide.
  const uint64_t magic = res_ld(ka.ctl), callno = res_ld(ka.ctl + 1);
  const bool fresh = magic != kResMagic;
  const int par = fresh ? 0 : static_cast<int>(callno & 1);
  uint64_t* reg = ka.region + static_cast<size_t>(par) * kResRegionWords;
  auto clear_region = [&](uint64_t* base) {
    constexpr size_t n2 = kResRegionWords / 2;
    const size_t per = (n2 + G - 1) / G, lo = static_cast<size_t>(g) * per, hi = min(n2, lo + per);
    for (size_t u = lo + threadIdx.x; u < hi; u += kResThreads) res_st2(base + 2 * u, kResEmpty, kResEmpty);
  };
  if (fresh) {
    clear_region(reg);
    cg::this_grid().sync();
  }
  clear_region(ka.region + static_cast<size_t>(par ^ 1) * kResRegionWords);
  uint64_t* const norms = reg;
  auto hdr = [&](int s, int q) { return reg + kResMaxG + (static_cast<size_t>(s) * kResMaxG + q) * 2; };
  auto rec = [&](int s, int q) {
    return reg + kResMaxG + kResHdrWords + (static_cast<size_t>(s) * kResMaxG + q) * kResRec;
  };

  // ---- load: row thread lr owns local rows lr + k * kResRowThreads (k < kResRPT) ----
  double xr[kResRPT][KR];
  bool live[kResRPT], has[kResRPT];
#pragma unroll
  for (int k = 0; k < kResRPT; ++k) {
    const int l = lr + k * kResRowThreads;
    has[k] = warp > 0 && l < nr;
    live[k] = false;
    if (has[k]) {
      const double* src = a.W + r0 + l;
      double* w = Ws + l;
#pragma unroll 8
      for (int t = 0; t < R0; ++t) w[t * ldS] = src[t * ldw];
#pragma unroll
      for (int j = 0; j < KR; ++j) xr[k][j] = R0 + j < steps ? src[(R0 + j) * ldw] : 0.0;
      const uint8_t mk = a.mask[r0 + l];
      live[k] = !(mk == 1 || mk == a.epoch);
    } else {
#pragma unroll
      for (int j = 0; j < KR; ++j) xr[k][j] = 0.0;
    }
  }
  const bool need_norm = a.d_norm_sq == nullptr;
  if (need_norm) {  // ||W(:, 0:steps)||_F^2: this CTA's partial, published for every CTA
    double sq = 0.0;
#pragma unroll
    for (int k = 0; k < kResRPT; ++k)
      if (has[k]) {
        const double* w = Ws + lr + k * kResRowThreads;
        for (int t = 0; t < R0; ++t) sq = fma(w[t * ldS], w[t * ldS], sq);
#pragma unroll
        for (int j = 0; j < KR; ++j)
          if (R0 + j < steps) sq = fma(xr[k][j], xr[k][j], sq);
      }
    const double b = block_sum<kResThreads>(sq, s_red);
    if (threadIdx.x == 0) res_st(norms + g, res_enc(b));
  }

#ifdef ITERCUR_RES_TRACE
  long long* const dbg = (ka.dbg && g == 0) ? ka.dbg : nullptr;
#else
  constexpr long long* dbg = nullptr;
#endif
  const int backoff = ka.backoff_ns;
  // ---- the exchange (warp 0): step s's CTA headers -> winner; its record -> the pivot row
  //      Pr[s % ring], its reciprocal and the runner-up ----
  auto exchange = [&](int s) {
    const uint64_t t0 = res_now();
    bool timed_out = false;
    auto wait = [&](uint64_t& spins) {
      if ((++spins & 255) == 0 && res_now() - t0 > kResTimeoutNs) timed_out = true;
      if (backoff) __nanosleep(backoff);
      return !timed_out;
    };
    // every header of the step polled at once (one L2 round trip when they are all there; a lane
    // re-polls only its missing ones); headers carry (key, row) only: the CTA keys give the winner
    // and the runner-up among CTA winners, the winning CTA's own runner-up is read with its row
    constexpr int QN = (kResMaxG + 31) / 32;
    unsigned pending = 0;
#pragma unroll
    for (int u = 0; u < QN; ++u)
      if (lane + 32 * u < G) pending |= 1u << u;
    WCand c{0ull, 0x7fffffff, -1.0};
    uint64_t spins = 0;
    while (true) {
      uint64_t k[QN], ix[QN];
#pragma unroll
      for (int u = 0; u < QN; ++u)
        if (pending >> u & 1) res_ld2(hdr(s, lane + 32 * u), k[u], ix[u]);
#pragma unroll
      for (int u = 0; u < QN; ++u)
        if ((pending >> u & 1) && k[u] != kResEmpty && ix[u] != kResEmpty) {
          pending &= ~(1u << u);
          wcand_merge(c, k[u], static_cast<int32_t>(ix[u]), -1.0);
        }
      if (!pending || !wait(spins)) break;
    }
    WCand best = warp_argmax(c);
    if (dbg && lane == 0) dbg[s * 8 + 6] = clock64();
#ifdef ITERCUR_RES_TRACE
    if (ka.gdbg && lane == 0) ka.gdbg[(static_cast<size_t>(s) * G + g) * 4 + 1] = static_cast<long long>(res_now());
#endif
    double* Pn = Pr[s & (kResRing - 1)];
    double y = 0.0;
    if (best.key) {  // word 2: the winning CTA's runner-up key; 4 + t: the row
      // RN(1/|pivot|) from the header's key while the row is in flight (RN(1/-p) = -RN(1/p))
      const double yabs = lane == 0 ? __drcp_rn(key_mag(best.key)) : 0.0;
      const uint64_t* wr = rec(s, static_cast<int>(best.idx / Rb));
      const int t0 = s + lane, t1 = s + lane + 32;
      uint64_t u0 = 0, u1 = 0, uh0 = 0;
      bool w0 = t0 < steps, w1 = t1 < steps, wh = lane == 0;
      spins = 0;
      while (true) {
        if (w0) u0 = res_ld(wr + 4 + t0);
        if (w1) u1 = res_ld(wr + 4 + t1);
        if (wh) uh0 = res_ld(wr + 2);
        w0 = w0 && u0 == kResEmpty;
        w1 = w1 && u1 == kResEmpty;
        wh = wh && uh0 == kResEmpty;
        if (!(w0 || w1 || wh) || !wait(spins)) break;
      }
      if (t0 < steps) Pn[t0] = __longlong_as_double(static_cast<long long>(u0));
      if (t1 < steps) Pn[t1] = __longlong_as_double(static_cast<long long>(u1));
      if (lane == 0) {
        if (uh0) best.second = fmax(best.second, key_mag(uh0));
        y = (u0 >> 63) ? -yabs : yabs;  // lane 0 holds column s: the pivot itself
      }
    }
    if (s == 0 && need_norm) {  // the CTA partials in a fixed tree: every CTA forms the same sum
      uint64_t nv[QN];
      unsigned pn = 0;
#pragma unroll
      for (int u = 0; u < QN; ++u)
        if (lane + 32 * u < G) pn |= 1u << u;
      spins = 0;
      while (true) {
#pragma unroll
        for (int u = 0; u < QN; ++u)
          if (pn >> u & 1) nv[u] = res_ld(norms + lane + 32 * u);
#pragma unroll
        for (int u = 0; u < QN; ++u)
          if ((pn >> u & 1) && nv[u] != kResEmpty) pn &= ~(1u << u);
        if (!pn || !wait(spins)) break;
      }
      double v = 0.0;
#pragma unroll
      for (int u = 0; u < QN; ++u)
        if (lane + 32 * u < G) v += __longlong_as_double(static_cast<long long>(nv[u]));
      v = warp_sum(v);
      if (lane == 0) s_nsq = v;
    }
    const bool abort = __any_sync(0xffffffffu, timed_out);
    if (dbg && lane == 0) dbg[s * 8 + 7] = clock64();
#ifdef ITERCUR_RES_TRACE
    if (ka.gdbg && lane == 0) ka.gdbg[(static_cast<size_t>(s) * G + g) * 4 + 2] = static_cast<long long>(res_now());
#endif
    if (lane == 0) {
      s_best = best;
      s_y = y;
      s_abort = abort ? 1 : 0;
      if (abort) atomicExch(reinterpret_cast<unsigned long long*>(ka.ctl + 2), 1ull);
    }
  };
  // ---- record sp of this CTA (warp 0, after [B2]): the CTA winner over the row warps' winners;
  //      header (key, row); runner-up and RN(1/value); the winner's row, current: shared-memory
  //      columns with the open panel's terms p0..pe in step order, register columns and the
  //      next-column value as its warp staged them ----
  auto publish = [&](int sp) {
    const WCand c = lane < kResWarps ? wc[lane] : WCand{0ull, 0x7fffffff, -1.0};
    const WCand cb = warp_argmax(c);
    if (dbg && lane == 0 && sp > 0) dbg[(sp - 1) * 8 + 2] = clock64() + (cb.key & 0);
    uint64_t* r = rec(sp, g);
    if (cb.key) {
      const int olr = static_cast<int>(cb.idx - r0), w = (olr % kResRowThreads) / 32 + 1;
      const double* orow = Ws + olr;
      if (lane == 0) res_st2(hdr(sp, g), cb.key, static_cast<uint64_t>(cb.idx));
      if (lane == 1) res_st(r + 2, cb.second >= 0.0 ? mag_key(cb.second) : 0ull);
      // the row, a lane per column; a shared-memory column t > sp owes its pending steps
      // j0..sp-1 (res_last_update(t, sp - 1) + 1 = sp - 1 - ((sp - 2 - t) mod kResPanel), >= 0),
      // at most kResPanel of them, their operands loaded together
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int t = sp + lane + 32 * h;
        if (t >= steps) continue;
        double v;
        if (t == sp) {
          v = stage[w][KR + 1];
        } else if (t < R0) {
          const int j0 = max(0, sp - 1 - ((sp - 2 - t) & (kResPanel - 1)));
          double mq[kResPanel], pq[kResPanel];
#pragma unroll
          for (int q = 0; q < kResPanel; ++q) {
            const int j = min(j0 + q, sp - 1 < 0 ? 0 : sp - 1);
            mq[q] = orow[j * ldS];
            pq[q] = Pr[j & (kResRing - 1)][t];
          }
          v = orow[t * ldS];
#pragma unroll
          for (int q = 0; q < kResPanel; ++q)
            if (j0 + q < sp) v = __dsub_rn(v, __dmul_rn(mq[q], pq[q]));
        } else {  // register column: current through step sp - 2, step sp - 1's term owed
          v = stage[w][t - R0];
          if (sp > 0) v = __dsub_rn(v, __dmul_rn(stage[w][KR], Pr[(sp - 1) & (kResRing - 1)][t]));
        }
        res_st(r + 4 + t, res_enc(v));
      }
      if (dbg && lane == 0 && sp > 0) dbg[(sp - 1) * 8 + 3] = clock64();
    } else if (lane == 0) {
      res_st2(hdr(sp, g), 0ull, 0ull);
      res_st(r + 2, 0ull);
    }
#ifdef ITERCUR_RES_TRACE
    if (ka.gdbg && lane == 0) ka.gdbg[(static_cast<size_t>(sp) * G + g) * 4] = static_cast<long long>(res_now());
#endif
  };
  // row warps: this thread's candidate over its rows (ascending local row: ties keep the lower),
  // the warp argmax, and the warp winner's registers + next-column value staged for the publish
  double cur[kResRPT];
#pragma unroll
  for (int k = 0; k < kResRPT; ++k) cur[k] = 0.0;
  double fk[kResRPT];
#pragma unroll
  for (int k = 0; k < kResRPT; ++k) fk[k] = 0.0;
  auto warp_pick = [&]() {
    WCand mine{0ull, 0x7fffffff, -1.0};
#pragma unroll
    for (int k = 0; k < kResRPT; ++k)
      if (live[k]) mine = wcand_merge_row(mine, fabs(cur[k]), static_cast<int32_t>(r0 + lr + k * kResRowThreads));
    const WCand w = warp_argmax(mine);
    if (w.key) {
#pragma unroll
      for (int k = 0; k < kResRPT; ++k)
        if (live[k] && static_cast<int64_t>(w.idx) == r0 + lr + k * kResRowThreads) {
#pragma unroll
          for (int j = 0; j < KR; ++j) stage[warp][j] = xr[k][j];
          stage[warp][KR] = fk[k];
          stage[warp][KR + 1] = cur[k];
        }
    }
    if (lane == 0) wc[warp] = w;
  };

  // ---- step-0 candidates (column 0) ----
  if (warp > 0) {
#pragma unroll
    for (int k = 0; k < kResRPT; ++k)
      if (live[k]) cur[k] = R0 > 0 ? Ws[lr + k * kResRowThreads] : xr[k][0];
    warp_pick();
  } else if (lane == 0) {
    wc[0] = WCand{0ull, 0x7fffffff, -1.0};
  }
  __syncthreads();
  if (warp == 0) publish(0);

  double* lu_blk = a.lu_out ? a.lu_out + (a.d_lu_r ? *a.d_lu_r : 0) * a.lu_ld : nullptr;
  int count = 0;
  double first = 0.0, abs_floor = 0.0;
  for (int s = 0; s < steps; ++s) {
    if (warp == 0) exchange(s);
    __syncthreads();  // B1
    if (dbg && threadIdx.x == 0) dbg[s * 8 + 0] = clock64() + 0 * s_best.key;
    if (s_abort) break;
    if (s == 0) abs_floor = 1e2 * 2.220446049250313e-16 * sqrt(need_norm ? s_nsq : *a.d_norm_sq);
    const WCand best = s_best;
    const double bm = key_mag(best.key);
    if (best.key == 0 || bm <= abs_floor) break;
    if (s == 0)
      first = bm;
    else if (bm < a.pivot_floor * first)
      break;
    if (g == 0 && threadIdx.x == 0) {
      a.d_idx[s] = best.idx;
      a.d_best[s] = bm;
      a.d_second[s] = best.second;
    }
    ++count;
    const double* Pc = Pr[s & (kResRing - 1)];
    const bool mine_pivot = best.idx >= r0 && best.idx < r0 + nr;
#pragma unroll
    for (int k = 0; k < kResRPT; ++k)
      if (live[k] && r0 + lr + k * kResRowThreads == best.idx) {  // the pivot row retires; its
        live[k] = false;                                           // register columns for its LU row
        if (lu_blk) {
#pragma unroll
          for (int j = 0; j < KR; ++j) emit[j] = xr[k][j];
        }
      }
    if (s + 1 >= steps) {
      if (lu_blk && mine_pivot) {
        __syncthreads();
        if (warp == 0) {
          const int olr = static_cast<int>(best.idx - r0);
          for (int t = lane; t < steps; t += 32)
            lu_blk[s + t * a.lu_ld] = t >= s ? Pc[t] : (t < R0 ? Ws[olr + t * ldS] : emit[t - R0]);
        }
      }
      break;
    }
    if (warp > 0) {
      const double pivot = Pc[s], ys = s_y;
      const bool p_ok = pivot_in_range(pivot);
      const int t1 = s + 1, j1 = res_last_update(t1, s) + 1;  // column t1's pending steps j1..s
      // the next pivot column's pending terms before step s do not need f: formed first, beside
      // the division (at most kResPanel - 1 of them, loads issued together)
      double vpart[kResRPT];
#pragma unroll
      for (int k = 0; k < kResRPT; ++k) {
        vpart[k] = 0.0;
        if (!live[k] || t1 >= R0) continue;
        const double* w = Ws + lr + k * kResRowThreads;
        double m[kResPanel - 1], pv[kResPanel - 1];
#pragma unroll
        for (int q = 0; q < kResPanel - 1; ++q) {
          const int j = j1 + q < s ? j1 + q : s;
          m[q] = w[j * ldS];
          pv[q] = Pr[j & (kResRing - 1)][t1];
        }
        double v = w[t1 * ldS];
#pragma unroll
        for (int q = 0; q < kResPanel - 1; ++q)
          if (j1 + q < s) v = __dsub_rn(v, __dmul_rn(m[q], pv[q]));
        vpart[k] = v;
      }
#pragma unroll
      for (int k = 0; k < kResRPT; ++k) {
        if (!live[k]) continue;
        double* w = Ws + lr + k * kResRowThreads;
        const double f = div_by_pivot(cur[k], pivot, ys, p_ok);
        fk[k] = f;
        if (s < R0) {
          w[s * ldS] = f;
        } else {
#pragma unroll
          for (int j = 0; j < KR; ++j)
            if (R0 + j == s) xr[k][j] = f;
        }
        // the next pivot column, current through step s: a shared-memory column (its pending
        // steps, in step order) or a register column (the others receive step s after [B2])
        if (t1 < R0) {
          cur[k] = __dsub_rn(vpart[k], __dmul_rn(f, Pc[t1]));
        } else {
#pragma unroll
          for (int j = 0; j < KR; ++j)
            if (R0 + j == t1) {
              xr[k][j] = __dsub_rn(xr[k][j], __dmul_rn(f, Pc[t1]));
              cur[k] = xr[k][j];
            }
        }
      }
      warp_pick();
    }
    __syncthreads();  // B2
    if (dbg && threadIdx.x == 0) dbg[s * 8 + 1] = clock64() + 0 * wc[1].key;
    if (warp == 0) {
      publish(s + 1);
      // the update pass below rewrites shared-memory columns the record was read from
      asm volatile("bar.arrive 1, %0;\n" ::"r"(kResThreads) : "memory");
      // this CTA owns pivot s: its LU row (multipliers of steps < s, then the pivot row)
      if (lu_blk && mine_pivot) {
        const int olr = static_cast<int>(best.idx - r0);
        for (int t = lane; t < steps; t += 32)
          lu_blk[s + t * a.lu_ld] = t >= s ? Pc[t] : (t < R0 ? Ws[olr + t * ldS] : emit[t - R0]);
      }
    }
    if (dbg && threadIdx.x == 0) dbg[s * 8 + 5] = clock64();
    if (warp > 0) {
      asm volatile("bar.sync 1, %0;\n" ::"r"(kResThreads) : "memory");
      // step s's term for the register columns after s + 1, and the shared-memory columns
      // t = s + kResPanel, s + 2 kResPanel, ... brought current through step s (each column is
      // touched once per kResPanel steps with its pending terms; the work is spread evenly)
#pragma unroll
      for (int k = 0; k < kResRPT; ++k) {
        if (!live[k]) continue;
        const double f = fk[k];
#pragma unroll
        for (int j = 0; j < KR; ++j)
          if (R0 + j > s + 1) xr[k][j] = __dsub_rn(xr[k][j], __dmul_rn(f, Pc[R0 + j]));
        if (s + kResPanel >= R0) continue;  // no shared-memory column left to bring current
        double* w = Ws + lr + k * kResRowThreads;
        const int j0 = res_last_update(s + kResPanel, s) + 1;  // the same for every column updated now
        double fp[kResPanel];
        const double* pj[kResPanel];
#pragma unroll
        for (int q = 0; q < kResPanel; ++q) {
          const int j = j0 + q <= s ? j0 + q : s;
          fp[q] = w[j * ldS];
          pj[q] = Pr[j & (kResRing - 1)];
        }
        const int nt = s + 1 - j0;  // terms (<= kResPanel)
        int t = s + kResPanel;
        for (; t + kResPanel < R0; t += 2 * kResPanel) {  // two columns in flight
          double v0 = w[t * ldS], v1 = w[(t + kResPanel) * ldS];
#pragma unroll
          for (int q = 0; q < kResPanel; ++q)
            if (q < nt) {
              v0 = __dsub_rn(v0, __dmul_rn(fp[q], pj[q][t]));
              v1 = __dsub_rn(v1, __dmul_rn(fp[q], pj[q][t + kResPanel]));
            }
          w[t * ldS] = v0;
          w[(t + kResPanel) * ldS] = v1;
        }
        if (t < R0) {
          double v0 = w[t * ldS];
#pragma unroll
          for (int q = 0; q < kResPanel; ++q)
            if (q < nt) v0 = __dsub_rn(v0, __dmul_rn(fp[q], pj[q][t]));
          w[t * ldS] = v0;
        }
      }
    }
  }
  if (g == 0 && threadIdx.x == 0) {
    *a.d_count = count;
    if (a.d_width_out) *a.d_width_out = min(count, *a.d_width_cap);
    // every CTA read the control words before publishing its step-0 record, which this CTA
    // has seen: the next call may now use the other region
    res_st(ka.ctl + 1, fresh ? 1ull : callno + 1);
    res_st(ka.ctl, kResMagic);
  }
}

static cudaError_t try_lupp_resident(const LuppArgs& a, void* res_scratch, cudaStream_t st, int* grid_used) {
  static const bool off = env_flag("ITERCUR_LUPP_NO_RESIDENT");
  if (off || a.cols_max > kResMaxSteps || a.cols_max < 1 || a.rows < 1 || a.rows >= (1ll << 31) - 1)
    return cudaErrorNotSupported;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int G = std::min(sms, kResMaxG);
  const int64_t Rb = ceil_div(a.rows, static_cast<int64_t>(G));
  if (Rb > kResRPT * kResRowThreads) return cudaErrorNotSupported;
  G = static_cast<int>(ceil_div(a.rows, Rb));
  const int R0 = std::max(a.cols_max - kResKR, 0);
  const size_t smem = sizeof(double) * static_cast<size_t>(R0) * (Rb | 1);
  constexpr size_t kDynMax = 208 * 1024;
  if (smem > kDynMax) return cudaErrorNotSupported;
  const void* fn = reinterpret_cast<const void*>(lupp_resident_kernel<kResKR>);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDynMax));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kResThreads, smem);
  if (per_sm < 1 || per_sm * sms < G) return cudaErrorNotSupported;
  LuppResArgs ka;
  ka.a = a;
  ka.ctl = reinterpret_cast<uint64_t*>(res_scratch);
  ka.region = ka.ctl + 8;
  ka.rows_per_cta = static_cast<int>(Rb);
  ka.dbg = g_lupp_dbg;
  ka.gdbg = g_lupp_gdbg;
  static const int backoff = [] {
    const char* e = getenv("ITERCUR_RES_BACKOFF_NS");
    return e ? atoi(e) : 0;
  }();
  ka.backoff_ns = backoff;
  void* params[] = {&ka};
  if (grid_used) *grid_used = -(300000 + G);  // negative: emits the LU factors itself
  return cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kResThreads), params, smem, st);
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
static size_t lupp_scratch_base_bytes(int b) {
  return sizeof(Cand) * 2 * kMaxLuppGrid + sizeof(double) * kMaxLuppGrid +
         sizeof(double) * 2 * kMaxLuppGrid * static_cast<size_t>(b + 4) + 64;  // + the panel kernel's arrivals
}
// the resident kernel's control words and exchange regions first (a fixed offset for every call
// sharing the buffer), then the other kernels' slots
size_t lupp_scratch_bytes(int b) { return kResScratchBytes + lupp_scratch_base_bytes(b); }
// A freshly allocated scratch may hold anything (pool memory reused from other buffers): the
// resident kernel's control words and regions are set to the sentinel before first use.
cudaError_t lupp_scratch_init(void* scratch, cudaStream_t st) {
  return cudaMemsetAsync(scratch, 0xFF, kResScratchBytes, st);
}

void set_lupp_force_path(int path) { g_force_path = path; }
void set_lupp_debug_trace(long long* dbg) { g_lupp_dbg = dbg; }
void set_lupp_grid_trace(long long* gdbg) { g_lupp_gdbg = gdbg; }

cudaError_t run_lupp_with_scratch(const LuppArgs& a, void* scratch, cudaStream_t st, int* grid_used) {
  if (a.cols_max > 2048) return cudaErrorInvalidValue;
  char* const res_scratch = reinterpret_cast<char*>(scratch);
  char* sp = res_scratch + kResScratchBytes;
  Cand* cand = reinterpret_cast<Cand*>(sp);
  double* norm_part = reinterpret_cast<double*>(sp + sizeof(Cand) * 2 * kMaxLuppGrid);
  // the panel kernel's arrival counter (never cleared: each launch reads its base), then the
  // shared-memory kernel's publication slots
  unsigned long long* arrivals = reinterpret_cast<unsigned long long*>(norm_part + kMaxLuppGrid);
  double* pub = norm_part + kMaxLuppGrid + 8;
  const int steps = std::max(a.cols_max, 1);
  // cluster path (W fits in one thread-block cluster's shared memory)
  if (g_force_path == 0 || g_force_path == 1) {
    cudaError_t e = try_lupp_cluster_v2(a, st, grid_used);
    if (e != cudaErrorNotSupported) return e;
    e = try_lupp_cluster(a, st, grid_used);
    if (e != cudaErrorNotSupported) return e;
  }
  // on-chip resident grid path (slab in registers + shared memory, fence-free exchange)
  if (g_force_path == 0 || g_force_path == 4) {
    cudaError_t e = try_lupp_resident(a, res_scratch, st, grid_used);
    if (e != cudaErrorNotSupported || g_force_path == 4) return e;
  }
  // shared-memory-resident path: one CTA per SM, slab of rows_per_cta x steps doubles
  if (g_force_path == 0 || g_force_path == 2) {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // enough rows per CTA to amortise the per-step exchange (~300), at most one CTA per SM
    const int G = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sms, ceil_div(a.rows, 300))));
    const int Rb = static_cast<int>(ceil_div(a.rows, G));
    const size_t smem =
        sizeof(double) * (static_cast<size_t>(steps) * Rb + (2 + kLuppThreads / 32) * steps + Rb) + Rb + 16;
    if (smem <= kLuppSmemBudget) {
      static size_t attr = 0;
      if (smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(lupp_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kLuppSmemBudget));
        if (e != cudaSuccess) return e;
        attr = kLuppSmemBudget;
      }
      if (lupp_max_blocks(reinterpret_cast<const void*>(lupp_smem_kernel), smem) >= G) {
        static uint32_t gen = 0x80000000u;  // host-side generations (stage entries) keep bit 31 set
        LuppSmemArgs ka;
        ka.a = a;
        ka.pub = pub;
        ka.pub_stride = steps + 4;
        ka.norm_part = norm_part;
        ka.rows_per_cta = Rb;
        ka.gen = ++gen | 0x80000000u;
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
  LuppKernelArgs ka;
  ka.a = a;
  ka.cand = cand;
  ka.norm_part = norm_part;
  ka.dbg = g_lupp_dbg;
  // the panel kernel's per-step exchange: counted arrivals instead of a grid barrier
  // (A/B: ITERCUR_LUPP_GRIDSYNC=1 keeps cooperative-groups grid.sync)
  static const bool gridsync = env_flag("ITERCUR_LUPP_GRIDSYNC");
  ka.arrivals = gridsync ? nullptr : arrivals;
  void* params[] = {&ka};
  static const bool right_looking = env_flag("ITERCUR_LUPP_RIGHT_LOOKING");  // A/B switch
  if (!right_looking && steps <= 2048) {
    // panel-blocked grid kernel: the fewest rows per thread whose co-resident grid covers the
    // slab (occupancy per variant: they differ in registers)
    struct Variant {
      const void* fn;
      int rmax, pg;
    };
    static const Variant variants[4] = {{reinterpret_cast<const void*>(lupp_panel_kernel<1, 8>), 1, 8},
                                        {reinterpret_cast<const void*>(lupp_panel_kernel<2, 8>), 2, 8},
                                        {reinterpret_cast<const void*>(lupp_panel_kernel<4, 8>), 4, 8},
                                        {reinterpret_cast<const void*>(lupp_panel_kernel<8, 4>), 8, 4}};
    static size_t pattr[4] = {0, 0, 0, 0};
    for (int v = 0; v < 4; ++v) {
      const size_t psmem = sizeof(double) * (static_cast<size_t>(steps) * (1 + variants[v].pg) +
                                             static_cast<size_t>(variants[v].pg) * variants[v].rmax * kLuppThreads);
      if (psmem > 48 * 1024 && psmem > pattr[v]) {
        cudaError_t e = cudaFuncSetAttribute(variants[v].fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(psmem));
        if (e != cudaSuccess) return e;
        pattr[v] = psmem;
      }
      const int maxb = std::min(lupp_max_blocks(variants[v].fn, psmem), kMaxLuppGrid);
      const int64_t need = ceil_div(a.rows, static_cast<int64_t>(variants[v].rmax) * kLuppThreads);
      if (maxb <= 0 || need > maxb) continue;
      const int grid = static_cast<int>(std::max<int64_t>(1, need));
      if (grid_used) *grid_used = -(200000 + grid);  // negative: emits the LU factors itself
      return cudaLaunchCooperativeKernel(variants[v].fn, dim3(grid), dim3(kLuppThreads), params, psmem, st);
    }
  }
  const size_t smem = sizeof(double) * static_cast<size_t>(steps);
  const int64_t want = std::max<int64_t>(1, ceil_div(a.rows, kLuppThreads));  // one row per thread
  const int maxb = lupp_max_blocks(reinterpret_cast<const void*>(lupp_kernel), smem);
  int grid = static_cast<int>(std::min<int64_t>(want, std::min(maxb, kMaxLuppGrid)));
  if (grid_used) *grid_used = 1000000 + grid;
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(lupp_kernel), dim3(grid), dim3(kLuppThreads),
                                     params, smem, st);
}

// a kernel of this translation unit (module), for itercur_preload
const void* module_anchor_lupp() { return reinterpret_cast<const void*>(lupp_kernel); }

}  // namespace itercur_b200

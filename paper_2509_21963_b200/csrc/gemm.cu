// gemm.cu — tall-skinny FP64 DMMA GEMM with gather/in-place epilogues, the workhorse of
// the per-iteration stages of the incremental (block-LU / Schur) form of IterativeCUR
// (SURVEY.md A.7), replacing the reference's per-iteration Eigen products:
//   row residual  S_row = A(:,J_k) - L * Rt(:,J_k)           (proj/src/sketch.cpp:43-60)
//   new U block   U_k^T = A(I_k,:)^T - Rt^T * L(I_k,:)^T      (proj/src/pinv.cpp:94-111 rebuild)
//   Y downdate    Y^T -= Rt_k^T * Y(:,J_k)^T  in place         (proj/src/sketch.cpp:26-41)
//   verification  ||A(:,P) - L * Rt(:,P)||^2                   (proj/src/driver.cpp:169-190)
//   core export   block substitutions with the stored D_k factors
//
//   C (M x N) = base(M x N) + alpha * Aop(M x K) * B(K x N)
// Aop is M-contiguous (column-major, even ld) and streamed once; B is tiny and may be
// gathered through an index list (B(k,q) = B[k*bsk + idx[q]*bsn]) so the selected columns /
// rows never need a separate copy. The M and K dimensions are permuted inside each
// 16x8x8 DMMA so that every A and B fragment pair is one 16-byte shared load: logical rows
// (g, g+8) -> physical (2g, 2g+1), logical k (t, t+4) -> physical (2t, 2t+1). Tiles are
// staged with cp.async in a 4-deep ring. The CTA height (WARPS x 16 rows) is chosen per
// call so that every launch spreads over several CTAs per SM (these GEMMs are HBM-bound:
// intensity 2N/8 flop/B ~ the FP64 ridge), keeping all SMs streaming.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "gemm.h"

namespace itercur_b200 {

constexpr int kGemmKT = 16;          // k per stage
constexpr int kGemmStages = 4;
constexpr int kBPitch = kGemmKT + 2;  // doubles; 144 B rows -> conflict-free 16-B fragment loads

template <int NT, int WARPS>
struct GemmCfg {
  static constexpr int THREADS = WARPS * 32;
  static constexpr int BM = WARPS * 16;
  static constexpr int A_ELEMS = kGemmKT * BM;
  static constexpr int B_ELEMS = NT * 8 * kBPitch;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr int BYTES = kGemmStages * STAGE_ELEMS * 8;
  static_assert(THREADS * NT * 4 <= kGemmStages * STAGE_ELEMS, "split-K reduction buffer must fit the ring");
};

__device__ __forceinline__ void cp_async_16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int NT, int WARPS>
__device__ __forceinline__ void gemm_load_stage(const TsGemmParams& p, double* sA, double* sB, int64_t i0, int64_t k0,
                                                int64_t q0, int nvalid, int64_t K) {
  using Cfg = GemmCfg<NT, WARPS>;
  // A tile: [kGemmKT][BM], 16-byte chunks of two consecutive rows
  constexpr int A_CHUNKS = kGemmKT * Cfg::BM / 2;
  for (int c = threadIdx.x; c < A_CHUNKS; c += Cfg::THREADS) {
    const int kl = c / (Cfg::BM / 2), il = (c % (Cfg::BM / 2)) * 2;
    const int64_t k = k0 + kl, i = i0 + il;
    int bytes = 0;
    const double* src = p.A;
    if (k < K && i < p.M) {
      bytes = (i + 1 < p.M) ? 16 : 8;
      src = p.A + i + k * p.lda;
    }
    cp_async_16(sA + kl * Cfg::BM + il, src, bytes);
  }
  // B tile: [NT*8][kBPitch], element (k, q) -> sB[q * kBPitch + k]
  if (p.bsk == 1 && !p.b_idx && (p.bsn & 1) == 0 && (reinterpret_cast<uintptr_t>(p.B) & 15) == 0) {
    // k-contiguous B: 16-byte copies of (k, k+1) pairs (k0 is a multiple of 16)
    constexpr int B_PAIRS = NT * 8 * kGemmKT / 2;
    for (int e = threadIdx.x; e < B_PAIRS; e += Cfg::THREADS) {
      const int ql = e / (kGemmKT / 2), kl = (e % (kGemmKT / 2)) * 2;
      const int64_t k = k0 + kl;
      int bytes = 0;
      const double* src = p.B;
      if (k < K && ql < nvalid) {
        bytes = (k + 1 < K) ? 16 : 8;
        src = p.B + k + (q0 + ql) * p.bsn;
      }
      cp_async_16(sB + ql * kBPitch + kl, src, bytes);
    }
    return;
  }
  constexpr int B_ELEMS = NT * 8 * kGemmKT;
  for (int e = threadIdx.x; e < B_ELEMS; e += Cfg::THREADS) {
    const int ql = e / kGemmKT, kl = e % kGemmKT;
    const int64_t k = k0 + kl;
    const int64_t q = q0 + ql;
    int bytes = 0;
    const double* src = p.B;
    if (k < K && ql < nvalid) {
      bytes = 8;
      const int64_t col = p.b_idx ? p.b_idx[q] : q;
      src = p.B + k * p.bsk + col * p.bsn;
    }
    cp_async_8(sB + ql * kBPitch + kl, src, bytes);
  }
}


__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ub_stamp(const TsGemmParams& p, int slot) {
  if (p.dbg && blockIdx.x == 0 && blockIdx.z == 0 && threadIdx.x == 0) p.dbg[slot] = clock64();
}
__device__ __forceinline__ void cta_stamp(const TsGemmParams& p, int which) {
  if (p.dbg && threadIdx.x == 0) p.dbg[32 + 2 * (blockIdx.x * gridDim.z + blockIdx.z) + which] = gtimer();
}

// Split-K cluster reduction (when gridDim.z > 1) and the fused epilogue: base + alpha * acc
// written per out_mode, with the per-CTA sum of squares of C.
template <int NT, int WARPS>
__device__ __forceinline__ void ublock_epilogue(const TsGemmParams& p, double (&acc)[NT][4], const double (&bv)[NT][4],
                                                const double (&yv)[NT + 1][4], const double* s_lu, const double* s_yg,
                                                int64_t i0, int w);

// base(i, q) of the epilogue (loaded before the split-K exchange so its latency overlaps it)
__device__ __forceinline__ double gemm_base(const TsGemmParams& p, int64_t i, int64_t q) {
  switch (p.base_mode) {
    case kBaseGatherCols: return p.src[i + p.idx[q] * p.lds];
    case kBaseGatherRowsT: return p.src[p.idx[q] + i * p.lds];
    case kBaseContigCols: return p.src[i + (p.col0 + q) * p.lds];
    case kBaseInPlaceRowMajor: return p.C0[i * p.ldc0 + q];
    case kBaseIdentityCols: return (i == p.col0 + q) ? 1.0 : 0.0;
    default: return 0.0;
  }
}

// base values of this thread's C fragment (split 0 only): issued before the main loop when
// p.early_base (the gathers — A(I_k,:) rows at ~1 TB/s of 32-byte sectors — overlap the DMMA
// loop instead of following it), else in the epilogue
template <int NT>
__device__ __forceinline__ void gemm_load_base(const TsGemmParams& p, double (&bv)[NT][4], int64_t r0, int64_t q0,
                                               int nvalid) {
  const int t = threadIdx.x & 3;
  const bool finisher = blockIdx.z == 0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int dq = 0; dq < 2; ++dq)
#pragma unroll
      for (int dr = 0; dr < 2; ++dr) {
        const int ql = nt * 8 + 2 * t + dq;
        const int64_t i = r0 + dr;
        bv[nt][dr * 2 + dq] = (finisher && ql < nvalid && i < p.M) ? gemm_base(p, i, q0 + ql) : 0.0;
      }
}

// base values staged in shared memory by cp.async (BSM) instead of registers: the wide blocks'
// 4 NT base registers per thread would otherwise stay allocated through the whole kernel
template <int NT>
__device__ __forceinline__ const void* gemm_base_addr(const TsGemmParams& p, int64_t i, int64_t q) {
  switch (p.base_mode) {
    case kBaseGatherCols: return p.src + i + p.idx[q] * p.lds;
    case kBaseGatherRowsT: return p.src + p.idx[q] + i * p.lds;
    case kBaseContigCols: return p.src + i + (p.col0 + q) * p.lds;
    case kBaseInPlaceRowMajor: return p.C0 + i * p.ldc0 + q;
    default: return nullptr;
  }
}

template <int NT, int WARPS, bool UB = false, bool BSM = false>
__device__ __forceinline__ void gemm_epilogue(const TsGemmParams& p, double (&acc)[NT][4], double (&bv)[NT][4],
                                              double* gsm, int64_t i0, int64_t q0, int nvalid, int splits) {
  constexpr int THREADS = WARPS * 32;
  constexpr int W = NT * 8;
  constexpr int NTY = NT + 1;
  constexpr int YP = ((W + 15) / 16) * 16 + 8;
  __shared__ double red[WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t r0 = i0 + warp * 16 + 2 * g;
  // epilogue operands fetched before the split-K exchange (their latency overlaps it): the
  // base values, and for the U block the Y^T rows to downdate and D_k's factors / Y(:,J_k)
  const bool finisher = blockIdx.z == 0;
  double yv[NTY][4];
  double* sbase = gsm + NT * 4 * THREADS;  // BSM: [nt * 4 + v][THREADS], past the split-K buffer
  if constexpr (BSM) {
    __syncthreads();  // the ring's last stage may still be read by other warps
    if (finisher) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int dq = 0; dq < 2; ++dq)
#pragma unroll
          for (int dr = 0; dr < 2; ++dr) {
            const int ql = nt * 8 + 2 * t + dq;
            const int64_t i = r0 + dr;
            const bool in = ql < nvalid && i < p.M;
            const void* src = in ? gemm_base_addr<NT>(p, i, q0 + ql) : nullptr;
            double* dst = sbase + (nt * 4 + dr * 2 + dq) * THREADS + threadIdx.x;
            if (src)
              cp_async_8(dst, src, 8);
            else  // no base, outside the tile, or the identity (kBaseIdentityCols)
              *dst = (in && p.base_mode == kBaseIdentityCols && i == p.col0 + q0 + ql) ? 1.0 : 0.0;
          }
      cp_async_commit();
    }
  } else if (!p.early_base) {
    gemm_load_base<NT>(p, bv, r0, q0, nvalid);
  }
  double* s_lu = gsm + NT * 4 * THREADS;  // past the split-K exchange buffer
  double* s_yg = s_lu + W * W + W;  // (W reciprocals behind the LU block)
  if constexpr (UB) {
    if (finisher) {
      // D_k's LU factors and Y(:,J_k)^T staged by cp.async now (the ring is drained): their
      // latency overlaps the split-K exchange
      __syncthreads();
      const int64_t rr = p.ctl ? p.ctl->r : 0;
      const double* lu = p.lu + rr * p.ldd;
      for (int e = threadIdx.x; e < W * W; e += THREADS) {
        const int a = e % W, b = e / W;
        const bool in = a < nvalid && b < nvalid;
        cp_async_8(s_lu + e, in ? lu + a + b * p.ldd : lu, in ? 8 : 0);
      }
      for (int e = threadIdx.x; e < NTY * 8 * W; e += THREADS) {
        const int h = e / W, q = e % W;
        const bool in = q < nvalid && h < p.ycp;
        cp_async_8(s_yg + h * YP + q, in ? p.yg + h + q * p.ycp : p.yg, in ? 8 : 0);
      }
      cp_async_commit();
    }
    // the Y^T rows to downdate, prefetched while the block is narrow (b <= 32); wider blocks
    // (NT > 4) load them in the epilogue instead: their accumulators, base values and the
    // downdate's fragments would not fit the register file together
    if constexpr (NT <= 4) {
#pragma unroll
      for (int ny = 0; ny < NTY; ++ny)
#pragma unroll
        for (int dq = 0; dq < 2; ++dq)
#pragma unroll
          for (int dr = 0; dr < 2; ++dr) {
            const int h = ny * 8 + 2 * t + dq;
            const int64_t j = r0 + dr;
            yv[ny][dr * 2 + dq] = (finisher && h < p.ycp && j < p.M) ? p.y[j * p.ycp + h] : 0.0;
          }
    }
  }
  ub_stamp(p, 1);
  if (splits > 1) {
    // fixed-order reduction over the cluster: rank z publishes its fragments in its own
    // shared memory, rank 0 adds ranks 1..S-1 in order (deterministic for a given S)
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    __syncthreads();
    if (blockIdx.z != 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int v = 0; v < 4; ++v) gsm[(nt * 4 + v) * THREADS + threadIdx.x] = acc[nt][v];
    }
    cl.sync();
    if (blockIdx.z == 0) {
      for (int src = 1; src < splits; ++src) {
        const double* peer = cl.map_shared_rank(gsm, src);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[nt][v] += peer[(nt * 4 + v) * THREADS + threadIdx.x];
      }
    }
    cl.sync();
    if (blockIdx.z != 0) {
      cta_stamp(p, 1);
      return;
    }
  }
  if constexpr (UB) {
    ub_stamp(p, 2);
    cp_async_wait<0>();
    __syncthreads();
    // reciprocals of U's diagonal, behind the LU block
    if (threadIdx.x < W) s_lu[W * W + threadIdx.x] = threadIdx.x < nvalid ? __drcp_rn(s_lu[threadIdx.x * (W + 1)]) : 0.0;
    __syncthreads();
    ub_stamp(p, 3);
    ublock_epilogue<NT, WARPS>(p, acc, bv, yv, s_lu, s_yg, i0, nvalid);
    ub_stamp(p, 8);
    cta_stamp(p, 1);
    return;
  }

  ub_stamp(p, 2);
  if constexpr (BSM) cp_async_wait<0>();  // this thread's own base slots
  // ---------------- epilogue: physical rows (2g, 2g+1), columns (2t, 2t+1) ----------
  double sq = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int dq = 0; dq < 2; ++dq) {
      const int ql = nt * 8 + 2 * t + dq;
      if (ql >= nvalid) continue;
      const int64_t q = q0 + ql;
#pragma unroll
      for (int dr = 0; dr < 2; ++dr) {
        const int64_t i = r0 + dr;
        if (i >= p.M) continue;
        const double base = BSM ? sbase[(nt * 4 + dr * 2 + dq) * THREADS + threadIdx.x] : bv[nt][dr * 2 + dq];
        const double v = base + p.alpha * acc[nt][dr * 2 + dq];
        sq = fma(v, v, sq);
        if (p.out_mode == kOutColMajor) {
          p.C0[i + q * p.ldc0] = v;
          if (p.C1) p.C1[i + q * p.ldc1] = v;
        } else if (p.out_mode == kOutRowMajor) {
          p.C0[i * p.ldc0 + q] = v;
          if (p.Wc && q < p.wc_rows) p.Wc[i + q * p.ldwc] = v;
        }
      }
    }
  }
  if (p.norm_part) {
    sq = warp_sum(sq);
    if (lane == 0) red[warp] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < WARPS; ++w) s += red[w];
      p.norm_part[blockIdx.y * gridDim.x + blockIdx.x] = s;
    }
  }
  ub_stamp(p, 8);
  cta_stamp(p, 1);
}


// Fused U-block epilogue (see gemm.h). The C fragment of a warp holds rows (2g, 2g+1) x
// columns (nt*8 + 2t, +1): one row's w entries live in the 4 lanes of a quad, so the
// substitutions broadcast x[p] inside the quad with shuffles. The solved fragment is
// already the A operand of the downdate MMA (same physical k permutation as the main
// loop: logical k t <-> column 2t, t+4 <-> 2t+1), so Y^T -= X Yg^T runs on DMMA without
// leaving registers.
template <int NT, int WARPS>
__device__ __forceinline__ void ublock_epilogue(const TsGemmParams& p, double (&acc)[NT][4], const double (&bv)[NT][4],
                                                const double (&yv)[NT + 1][4], const double* s_lu, const double* s_yg,
                                                int64_t i0, int w) {
  constexpr int W = NT * 8;          // max block width
  constexpr int NTY = NT + 1;        // n-tiles of the downdate (ycp <= 8 * (NT + 1))
  constexpr int YP = ((W + 15) / 16) * 16 + 8;  // Yg^T pitch: 16-byte loads conflict-free
  __shared__ double red[WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t r = p.ctl ? p.ctl->r : 0;

  // u = base + alpha * acc (base = A(I_k[q], j), prefetched), zero outside the block
  const int64_t r0 = i0 + warp * 16 + 2 * g;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int dq = 0; dq < 2; ++dq) {
      const int q = nt * 8 + 2 * t + dq;
#pragma unroll
      for (int dr = 0; dr < 2; ++dr) {
        const int64_t j = r0 + dr;
        double v = 0.0;
        if (q < w && j < p.M) v = bv[nt][dr * 2 + dq] + p.alpha * acc[nt][dr * 2 + dq];
        acc[nt][dr * 2 + dq] = v;
      }
    }
  const int qbase = lane & ~3;
  if constexpr (NT > 4) {
    // wide blocks (33..64): the same substitutions as below with runtime loops over the pivot p
    // (the fully unrolled form outgrows the instruction cache at NT = 7: ncu showed "no
    // instruction" as the top stall and 785 us per call at config 4); x[p] is read from its
    // n-tile with a static select, so acc never needs a dynamic register index
    auto pick = [&](int ntp, int dqp, int row) {
      double v = 0.0;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        if (nt == ntp) v = dqp ? acc[nt][row * 2 + 1] : acc[nt][row * 2];
      return v;
    };
#pragma unroll 1
    for (int pp = 0; pp < w; ++pp) {
      const int ntp = pp >> 3, tp = (pp & 7) >> 1, dqp = pp & 1;
      const double x0 = __shfl_sync(0xffffffffu, pick(ntp, dqp, 0), qbase | tp);
      const double x1 = __shfl_sync(0xffffffffu, pick(ntp, dqp, 1), qbase | tp);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int dq = 0; dq < 2; ++dq) {
          const int q = nt * 8 + 2 * t + dq;
          if (q > pp && q < w) {
            const double l = s_lu[q + pp * W];
            acc[nt][dq] = fma(-l, x0, acc[nt][dq]);
            acc[nt][2 + dq] = fma(-l, x1, acc[nt][2 + dq]);
          }
        }
    }
    ub_stamp(p, 4);
#pragma unroll 1
    for (int pp = w - 1; pp >= 0; --pp) {
      const int ntp = pp >> 3, tp = (pp & 7) >> 1, dqp = pp & 1;
      const double upp = s_lu[pp + pp * W];
      const double a0 = __shfl_sync(0xffffffffu, pick(ntp, dqp, 0), qbase | tp);
      const double a1 = __shfl_sync(0xffffffffu, pick(ntp, dqp, 1), qbase | tp);
      const double yrc = s_lu[W * W + pp];
      double x0 = __dmul_rn(a0, yrc), x1 = __dmul_rn(a1, yrc);
      x0 = __fma_rn(__fma_rn(-x0, upp, a0), yrc, x0);
      x1 = __fma_rn(__fma_rn(-x1, upp, a1), yrc, x1);
      auto out_of_range = [](double v) {
        const unsigned hi = static_cast<unsigned>(__double_as_longlong(v) >> 32) & 0x7fffffffu;
        const unsigned e = hi >> 20;
        return static_cast<unsigned>((e - 56u) > (1990u - 56u)) & static_cast<unsigned>(v != 0.0);
      };
      const unsigned bad = out_of_range(a0) | out_of_range(a1) | out_of_range(x0) | out_of_range(x1) |
                           static_cast<unsigned>(!pivot_in_range(upp));
      if (__any_sync(0xffffffffu, bad)) {
        x0 = ieee_div(a0, upp);
        x1 = ieee_div(a1, upp);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        if (nt == ntp && t == tp) {
          if (dqp) {
            acc[nt][1] = x0;
            acc[nt][3] = x1;
          } else {
            acc[nt][0] = x0;
            acc[nt][2] = x1;
          }
        }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int dq = 0; dq < 2; ++dq) {
          const int q = nt * 8 + 2 * t + dq;
          if (q < pp) {
            const double u = s_lu[q + pp * W];
            acc[nt][dq] = fma(-u, x0, acc[nt][dq]);
            acc[nt][2 + dq] = fma(-u, x1, acc[nt][2 + dq]);
          }
        }
    }
  } else {
  // forward substitution with the unit-lower factor: x[q] -= L(q, p) x[p], p ascending
#pragma unroll
  for (int pp = 0; pp < W; ++pp) {
    if (pp >= w) break;
    const int ntp = pp / 8, tp = (pp % 8) / 2, dqp = pp % 2;
    const double x0 = __shfl_sync(0xffffffffu, acc[ntp][dqp], qbase | tp);
    const double x1 = __shfl_sync(0xffffffffu, acc[ntp][2 + dqp], qbase | tp);
#pragma unroll
    for (int nt = ntp; nt < NT; ++nt)
#pragma unroll
      for (int dq = 0; dq < 2; ++dq) {
        const int q = nt * 8 + 2 * t + dq;
        if (q > pp && q < w) {
          const double l = s_lu[q + pp * W];
          acc[nt][dq] = fma(-l, x0, acc[nt][dq]);
          acc[nt][2 + dq] = fma(-l, x1, acc[nt][2 + dq]);
        }
      }
  }
  ub_stamp(p, 4);
  // back substitution with U: x[p] /= U(p, p), then x[q] -= U(q, p) x[p] for q < p
#pragma unroll
  for (int pp = W - 1; pp >= 0; --pp) {
    if (pp >= w) continue;
    const int ntp = pp / 8, tp = (pp % 8) / 2, dqp = pp % 2;
    const double upp = s_lu[pp + pp * W];
    const double a0 = __shfl_sync(0xffffffffu, acc[ntp][dqp], qbase | tp);
    const double a1 = __shfl_sync(0xffffffffu, acc[ntp][2 + dqp], qbase | tp);
    // x = a / U(p, p) by Markstein's sequence from the precomputed reciprocal (the IEEE quotient
    // when a, x and U(p, p) lie inside [2^-968, 2^968] or a = 0); the IEEE division for the
    // whole warp otherwise (a warp-uniform branch keeps the chain short)
    const double yrc = s_lu[W * W + pp];
    double x0 = __dmul_rn(a0, yrc), x1 = __dmul_rn(a1, yrc);
    x0 = __fma_rn(__fma_rn(-x0, upp, a0), yrc, x0);
    x1 = __fma_rn(__fma_rn(-x1, upp, a1), yrc, x1);
    // in range: zero, or biased exponent in [56, 1990] (inside 2^-968 .. 2^968); branch-free
    auto out_of_range = [](double v) {
      const unsigned hi = static_cast<unsigned>(__double_as_longlong(v) >> 32) & 0x7fffffffu;
      const unsigned e = hi >> 20;
      return static_cast<unsigned>((e - 56u) > (1990u - 56u)) & static_cast<unsigned>(v != 0.0);
    };
    const unsigned bad = out_of_range(a0) | out_of_range(a1) | out_of_range(x0) | out_of_range(x1) |
                         static_cast<unsigned>(!pivot_in_range(upp));
    if (__any_sync(0xffffffffu, bad)) {
      x0 = ieee_div(a0, upp);
      x1 = ieee_div(a1, upp);
    }
    if (t == tp) {
      acc[ntp][dqp] = x0;
      acc[ntp][2 + dqp] = x1;
    }
#pragma unroll
    for (int nt = 0; nt <= ntp; ++nt)
#pragma unroll
      for (int dq = 0; dq < 2; ++dq) {
        const int q = nt * 8 + 2 * t + dq;
        if (q < pp) {
          const double u = s_lu[q + pp * W];
          acc[nt][dq] = fma(-u, x0, acc[nt][dq]);
          acc[nt][2 + dq] = fma(-u, x1, acc[nt][2 + dq]);
        }
      }
  }
  }
  ub_stamp(p, 5);
  // R~ rows r .. r+w
  double* rt = p.rt + r * p.ldr;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int dq = 0; dq < 2; ++dq) {
      const int q = nt * 8 + 2 * t + dq;
      if (q >= w) continue;
#pragma unroll
      for (int dr = 0; dr < 2; ++dr) {
        const int64_t j = r0 + dr;
        if (j < p.M) rt[q * p.ldr + j] = acc[nt][dr * 2 + dq];
      }
    }
  ub_stamp(p, 6);
  // downdate MMA: D(j, h) = sum_q x_j[q] Yg(h, q)
  double yacc[NTY][4];
#pragma unroll
  for (int ny = 0; ny < NTY; ++ny)
#pragma unroll
    for (int v = 0; v < 4; ++v) yacc[ny][v] = 0.0;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int ny = 0; ny < NTY; ++ny) {
      const double2 b = *reinterpret_cast<const double2*>(s_yg + (ny * 8 + g) * YP + nt * 8 + 2 * t);
      dmma_16x8x8(yacc[ny], acc[nt][0], acc[nt][2], acc[nt][1], acc[nt][3], b.x, b.y);
    }
  }
  double sq = 0.0;
#pragma unroll
  for (int ny = 0; ny < NTY; ++ny)
#pragma unroll
    for (int dq = 0; dq < 2; ++dq) {
      const int h = ny * 8 + 2 * t + dq;
      if (h >= p.ycp) continue;
#pragma unroll
      for (int dr = 0; dr < 2; ++dr) {
        const int64_t j = r0 + dr;
        if (j >= p.M) continue;
        const double y0 = NT <= 4 ? yv[ny][dr * 2 + dq] : p.y[j * p.ycp + h];
        const double v = y0 + p.alpha * yacc[ny][dr * 2 + dq];
        p.y[j * p.ycp + h] = v;
        sq = fma(v, v, sq);
        if (h < p.wc_rows) p.Wc[j + h * p.ldwc] = v;
      }
    }
  ub_stamp(p, 7);
  sq = warp_sum(sq);
  if (lane == 0) red[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < WARPS; ++q) s += red[q];
    p.norm_part[blockIdx.x] = s;
  }
  if (p.commit.ctl) {
    // the last finishing CTA commits the iteration (replaces the commit kernel's launch): every
    // CTA's partial is published before its arrival, so the fixed-order sum sees all of them
    __shared__ int s_last;
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(p.commit.counter, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      commit_body<WARPS * 32>(p.commit, p.norm_part, gridDim.x, red);
      if (threadIdx.x == 0) *p.commit.counter = 0;
    }
  }
}

// fused U block: n-tiles of 8 for blocks up to 64 wide
static int ts_gemm_nt_host(int n) { return n <= 64 ? static_cast<int>(std::max<int64_t>(1, ceil_div(n, 8))) : 9; }

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int NT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) ts_gemm_kernel(TsGemmParams p) {
  using Cfg = GemmCfg<NT, WARPS>;
  extern __shared__ __align__(16) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  griddep_wait();
  if (p.ctl) {
    if (p.ctl->done) return;
    const int64_t r = p.ctl->r;
    if (p.k_from_r) p.K = min(p.K, r);
    p.A += r * p.a_off_per_r;
    p.C0 += r * p.c0_off_per_r;
  }
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * Cfg::BM;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * (NT * 8);
  int n_total = p.N;
  if (p.d_n) n_total = min(n_total, *p.d_n);
  int64_t nv = static_cast<int64_t>(n_total) - q0;
  nv = nv < 0 ? 0 : (nv > NT * 8 ? NT * 8 : nv);
  const int nvalid = static_cast<int>(nv);

  double acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[nt][v] = 0.0;

  int64_t K = p.K;
  if (p.d_k) K = min(K, static_cast<int64_t>(*p.d_k));
  // split-K: the CTAs of one (1, 1, S) cluster share the output tile and take consecutive
  // ranges of k-stages; partial accumulators are summed in rank order through DSMEM below.
  const int nk_all = nvalid > 0 ? static_cast<int>(ceil_div(K, kGemmKT)) : 0;
  const int splits = static_cast<int>(gridDim.z);
  const int per_split = (nk_all + splits - 1) / splits;
  const int kb = static_cast<int>(blockIdx.z) * per_split;
  const int nk = max(0, min(nk_all - kb, per_split));
  const int64_t kbase = static_cast<int64_t>(kb) * kGemmKT;
  double bv[NT][4];
  if (p.early_base) gemm_load_base<NT>(p, bv, i0 + warp * 16 + 2 * g, q0, nvalid);
#pragma unroll
  for (int s = 0; s < kGemmStages - 1; ++s) {
    if (s < nk)
      gemm_load_stage<NT, WARPS>(p, gsm + s * Cfg::STAGE_ELEMS, gsm + s * Cfg::STAGE_ELEMS + Cfg::A_ELEMS, i0,
                                 kbase + static_cast<int64_t>(s) * kGemmKT, q0, nvalid, K);
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<kGemmStages - 2>();
    __syncthreads();
    const int nxt = it + kGemmStages - 1;
    if (nxt < nk) {
      double* base = gsm + (nxt % kGemmStages) * Cfg::STAGE_ELEMS;
      gemm_load_stage<NT, WARPS>(p, base, base + Cfg::A_ELEMS, i0, kbase + static_cast<int64_t>(nxt) * kGemmKT, q0,
                                 nvalid, K);
    }
    cp_async_commit();
    const double* sA = gsm + (it % kGemmStages) * Cfg::STAGE_ELEMS;
    const double* sB = sA + Cfg::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < kGemmKT; kk += 8) {
      const int rb = warp * 16 + 2 * g;
      const double2 a01 = *reinterpret_cast<const double2*>(sA + (kk + 2 * t) * Cfg::BM + rb);
      const double2 a23 = *reinterpret_cast<const double2*>(sA + (kk + 2 * t + 1) * Cfg::BM + rb);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double2 b = *reinterpret_cast<const double2*>(sB + (nt * 8 + g) * kBPitch + kk + 2 * t);
        dmma_16x8x8(acc[nt], a01.x, a01.y, a23.x, a23.y, b.x, b.y);
      }
    }
  }
  cp_async_wait<0>();
  griddep_launch_dependents();
  gemm_epilogue<NT, WARPS>(p, acc, bv, gsm, i0, q0, nvalid, splits);
}


// ---------------------------------------------------------------------------------
// Lean main loop for the hot shapes (row residual, U block, verification): Aop 16-byte
// aligned with even lda, B k-contiguous (bsk == 1, even bsn). Every thread's cp.async
// sources are fixed offsets from two per-thread base pointers, so a stage costs a handful
// of instructions per thread (the generic loader spends ~10x more on index math). Padded
// shared rows make every 16-byte fragment load conflict-free:
//   A stage [KT][BM + 2]: lane (g, t) reads chunk 2t*(BM+2)/2 + g = t*(BM+2) + g -> 8 banks
//   B stage [NT*8][KT + 8]: row pitch (KT+8)/2 chunks = 4 (mod 8) separates g from g+1
// ---------------------------------------------------------------------------------
template <int NT, int WARPS, int KT, int STAGES>
struct LeanCfg {
  static constexpr int THREADS = WARPS * 32;
  static constexpr int BM = WARPS * 16;
  static constexpr int AP = BM + 2;  // A row pitch (doubles)
  static constexpr int BP = KT + 8;  // B row pitch (doubles)
  static constexpr int A_ELEMS = KT * AP;
  static constexpr int B_ELEMS = NT * 8 * BP;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr int BYTES = STAGES * STAGE_ELEMS * 8;
  static constexpr int A_KSTEP = THREADS / (BM / 2);  // k rows covered per pass (= 4)
  static constexpr int A_PER = KT / A_KSTEP;
  static constexpr int B_QSTEP = THREADS / (KT / 2);  // q columns covered per pass
  static constexpr int B_PER = (NT * 8 + B_QSTEP - 1) / B_QSTEP;
  static_assert(THREADS % (BM / 2) == 0 && KT % A_KSTEP == 0, "A tiling");
  static_assert(THREADS % (KT / 2) == 0, "B tiling");
  static_assert(THREADS * NT * 4 <= STAGES * STAGE_ELEMS, "split-K reduction buffer must fit the ring");
};

template <int NT, int WARPS, int KT, int STAGES, bool UB = false, bool BSM = false>
__global__ void __launch_bounds__(WARPS * 32) ts_gemm_lean_kernel(TsGemmParams p) {
  using Cfg = LeanCfg<NT, WARPS, KT, STAGES>;
  extern __shared__ __align__(16) double gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  griddep_wait();
  if (p.dbg) {
    if (p.ctl && p.ctl->k != p.dbg_k) p.dbg = nullptr;
    cta_stamp(p, 0);
    ub_stamp(p, 0);
  }
  if (p.ctl) {
    if (p.ctl->done) return;
    const int64_t r = p.ctl->r;
    if (p.k_from_r) p.K = min(p.K, r);
    p.A += r * p.a_off_per_r;
    p.C0 += r * p.c0_off_per_r;
  }
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * Cfg::BM;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * (NT * 8);
  int n_total = p.N;
  if (p.d_n) n_total = min(n_total, *p.d_n);
  int64_t nv = static_cast<int64_t>(n_total) - q0;
  nv = nv < 0 ? 0 : (nv > NT * 8 ? NT * 8 : nv);
  const int nvalid = static_cast<int>(nv);
  int64_t K = p.K;
  if (p.d_k) K = min(K, static_cast<int64_t>(*p.d_k));

  const int nk_all = nvalid > 0 ? static_cast<int>(ceil_div(K, KT)) : 0;
  const int splits = static_cast<int>(gridDim.z);
  const int per_split = (nk_all + splits - 1) / splits;
  const int kb = static_cast<int>(blockIdx.z) * per_split;
  const int nk = max(0, min(nk_all - kb, per_split));

  // per-thread load descriptors
  const int a_il = (threadIdx.x % (Cfg::BM / 2)) * 2;
  const int a_kl0 = threadIdx.x / (Cfg::BM / 2);
  const int64_t a_row = i0 + a_il;
  const int a_bytes = a_row + 1 < p.M ? 16 : (a_row < p.M ? 8 : 0);
  const double* a_src = p.A + (a_row < p.M ? a_row : 0) + static_cast<int64_t>(a_kl0) * p.lda;
  const int64_t a_kstride = static_cast<int64_t>(Cfg::A_KSTEP) * p.lda;
  const uint32_t a_dst = smem_u32(gsm) + static_cast<uint32_t>((a_kl0 * Cfg::AP + a_il) * 8);
  const int b_kl = (threadIdx.x % (KT / 2)) * 2;
  const int b_ql0 = threadIdx.x / (KT / 2);
  const double* b_src = p.B + b_kl + (q0 + b_ql0) * p.bsn;
  const int64_t b_qstride = static_cast<int64_t>(Cfg::B_QSTEP) * p.bsn;
  const uint32_t b_dst = smem_u32(gsm) + static_cast<uint32_t>((Cfg::A_ELEMS + b_ql0 * Cfg::BP + b_kl) * 8);

  auto load = [&](int stage_slot, int kstage) {
    const int64_t k0 = static_cast<int64_t>(kstage) * KT;
    const bool full = k0 + KT <= K;
    const uint32_t so = static_cast<uint32_t>(stage_slot * Cfg::STAGE_ELEMS * 8);
    const double* as = a_src + k0 * p.lda;
#pragma unroll
    for (int j = 0; j < Cfg::A_PER; ++j) {
      const int kl = a_kl0 + j * Cfg::A_KSTEP;
      const int bytes = (full || k0 + kl < K) ? a_bytes : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                       a_dst + so + static_cast<uint32_t>(j * Cfg::A_KSTEP * Cfg::AP * 8)),
                   "l"(as + j * a_kstride), "r"(bytes)
                   : "memory");
    }
    const double* bs = b_src + k0;
#pragma unroll
    for (int j = 0; j < Cfg::B_PER; ++j) {
      const int ql = b_ql0 + j * Cfg::B_QSTEP;
      if (Cfg::B_PER * Cfg::B_QSTEP == NT * 8 || ql < NT * 8) {
        const int64_t k = k0 + b_kl;
        const int bytes = ql < nvalid ? ((full || k + 1 < K) ? 16 : (k < K ? 8 : 0)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                         b_dst + so + static_cast<uint32_t>(j * Cfg::B_QSTEP * Cfg::BP * 8)),
                     "l"(bytes ? bs + j * b_qstride : p.B), "r"(bytes)
                     : "memory");
      }
    }
  };

  double acc[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[nt][v] = 0.0;

  double bv[NT][4];
  if (!BSM && p.early_base) gemm_load_base<NT>(p, bv, i0 + warp * 16 + 2 * g, q0, nvalid);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, kb + s);
    cp_async_commit();
  }
  const int rb = warp * 16 + 2 * g;
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = it + STAGES - 1;
    if (nxt < nk) load(nxt % STAGES, kb + nxt);
    cp_async_commit();
    const double* sA = gsm + (it % STAGES) * Cfg::STAGE_ELEMS;
    const double* sB = sA + Cfg::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < KT; kk += 8) {
      const double2 a01 = *reinterpret_cast<const double2*>(sA + (kk + 2 * t) * Cfg::AP + rb);
      const double2 a23 = *reinterpret_cast<const double2*>(sA + (kk + 2 * t + 1) * Cfg::AP + rb);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double2 b = *reinterpret_cast<const double2*>(sB + (nt * 8 + g) * Cfg::BP + kk + 2 * t);
        dmma_16x8x8(acc[nt], a01.x, a01.y, a23.x, a23.y, b.x, b.y);
      }
    }
  }
  cp_async_wait<0>();
  griddep_launch_dependents();
  gemm_epilogue<NT, WARPS, UB, BSM>(p, acc, bv, gsm, i0, q0, nvalid, splits);
}

// CTA height: 64 rows (4 warps) unless overridden; measured best across the row-residual,
// U-block and downdate shapes (tools/bench_gemm.py).
static int gemm_warps(int64_t) {
  static const int forced = env_int("ITERCUR_GEMM_WARPS", 0);  // tuning override: 2, 4 or 8
  if (forced == 2 || forced == 4 || forced == 8) return forced;
  return 4;
}

// split-K factor: enough CTAs for ~4 resident per SM, each split keeping >= 4 k-stages.
static thread_local int g_splits_override = 0;  // per-launch override (U block tuning)
static int gemm_splits(int64_t tiles, int64_t K, int kt) {
  static const int forced_env = env_int("ITERCUR_GEMM_SPLITS", 0);
  const int forced = g_splits_override > 0 ? g_splits_override : forced_env;
  const int64_t stages = ceil_div(K, kt);
  int s = forced > 0 ? forced : static_cast<int>(ceil_div(4 * kNumSMs, std::max<int64_t>(tiles, 1)));
  // a split must own >= 10 k-stages: below that one wave of unsplit CTAs is faster (row-residual
  // shape 20000 x 20, B200: K = 400 -> 26.8 us unsplit vs 28.9 at 2 splits; K = 1600 -> 86 vs 76)
  s = static_cast<int>(std::min<int64_t>(s, std::max<int64_t>(1, stages / 10)));
  return std::max(1, std::min(s, 8));
}

static thread_local bool g_plan_only = false;  // ts_gemm_planned_splits: compute the grid, do not launch
static thread_local int g_planned_z = 0;
template <typename Kern>
static cudaError_t launch_split(Kern kern, dim3 grid, int threads, int bytes, const TsGemmParams& p, cudaStream_t st) {
  g_planned_z = static_cast<int>(grid.z);
  if (g_plan_only) return cudaSuccess;
  return launch_ex(kern, grid, dim3(threads), bytes, st, dim3(grid.z > 1 ? 1 : 0, 1, grid.z), p);
}

template <int NT, int WARPS>
static cudaError_t launch_cfg(const TsGemmParams& p, cudaStream_t st) {
  using Cfg = GemmCfg<NT, WARPS>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(ts_gemm_kernel<NT, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(p.M, Cfg::BM)), static_cast<unsigned>(ceil_div(p.N, NT * 8)));
  grid.z = static_cast<unsigned>(gemm_splits(static_cast<int64_t>(grid.x) * grid.y, p.k_plan > 0 ? p.k_plan : p.K, kGemmKT));
  return launch_split(ts_gemm_kernel<NT, WARPS>, grid, Cfg::THREADS, Cfg::BYTES, p, st);
}

template <int NT, int WARPS, int KT, int STAGES, bool UB = false, bool BSM = false>
static cudaError_t launch_lean(const TsGemmParams& p, cudaStream_t st) {
  using Cfg = LeanCfg<NT, WARPS, KT, STAGES>;
  static_assert(!BSM || 2 * NT * 4 * Cfg::THREADS <= STAGES * Cfg::STAGE_ELEMS, "base slots must fit the ring");
  static_assert(!UB || (NT * 4 * Cfg::THREADS + NT * 8 * NT * 8 + NT * 8 + (NT + 1) * 8 * (((NT * 8 + 15) / 16) * 16 + 8) <=
                        STAGES * Cfg::STAGE_ELEMS), "U-block epilogue buffers must fit the ring");
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(ts_gemm_lean_kernel<NT, WARPS, KT, STAGES, UB, BSM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(static_cast<unsigned>(ceil_div(p.M, Cfg::BM)), static_cast<unsigned>(ceil_div(p.N, NT * 8)));
  grid.z = static_cast<unsigned>(gemm_splits(static_cast<int64_t>(grid.x) * grid.y, p.k_plan > 0 ? p.k_plan : p.K, KT));
  return launch_split(ts_gemm_lean_kernel<NT, WARPS, KT, STAGES, UB, BSM>, grid, Cfg::THREADS, Cfg::BYTES, p, st);
}

// lean main loop eligibility: 16-byte aligned A rows pairs (even lda and offsets), k-contiguous B
static bool lean_ok(const TsGemmParams& p) {
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  return p.bsk == 1 && !p.b_idx && (p.bsn & 1) == 0 && al16(p.B) && al16(p.A) && (p.lda & 1) == 0 &&
         (p.a_off_per_r & 1) == 0;
}

template <int NT>
static cudaError_t launch_nt(const TsGemmParams& p, cudaStream_t st) {
  // 0 off, 1: KT16 x4, 2: KT32 x3, 3: KT32 x4, 4: KT16 x3, 5: KT32 x2; default by shape
  // (tools/time_stage.py gemm sweeps on B200: the lean loop wins for N <= 32 (KT32 x3 for the
  // taller M); for 33..72-wide blocks KT16 x3 / KT32 x2 beat the generic loop by 25-35%, e.g.
  // 100000 x 50 x 256: 130 vs 201 us, 200000 x 64 x 1024: 958 vs 1193 us; with the base values
  // staged in shared memory (128 instead of 168 registers) KT32 x2 reaches 125 / 882 us)
  static const int forced = env_int("ITERCUR_GEMM_LEAN", -1);
  const int64_t kp = p.k_plan > 0 ? p.k_plan : p.K;
  // (the U block's scattered A(I_k, :) base: KT16 x3 — 201 vs 246 us per call at config 4; the
  // in-place downdate: KT32 x2 — 43 vs 50 us at config 5; per-role times: tools/gemm_roles.py)
  const bool gather_rows = p.base_mode == kBaseGatherRowsT;
  const bool kt32 = (kp >= 256 || p.base_mode == kBaseInPlaceRowMajor) && !gather_rows;
  const int lean = forced >= 0 ? forced : (NT > 4 ? (kt32 ? 5 : 4) : (p.M >= 16000 ? 2 : 1));
  if (lean > 0 && lean_ok(p) && gemm_warps(p.M) == 4) {
    // wide blocks without early base loads: base values staged through shared memory (A/B:
    // ITERCUR_GEMM_BSM=0) — except the U block's scattered A(I_k, :) gather, whose 8-byte cp.asyncs
    // ran slower than register loads (ncu, config 4: 226 vs 173 us)
    static const int bsm_env_raw = env_int("ITERCUR_GEMM_BSM", 1);
    const int bsm_env = bsm_env_raw && !gather_rows;
    constexpr bool fit4 = 2 * NT * 4 * 128 <= 3 * LeanCfg<NT, 4, 16, 3>::STAGE_ELEMS;
    constexpr bool fit5 = 2 * NT * 4 * 128 <= 2 * LeanCfg<NT, 4, 32, 2>::STAGE_ELEMS;
    if constexpr (NT > 4 && fit4) {
      if (bsm_env && !p.early_base && lean == 4) return launch_lean<NT, 4, 16, 3, false, true>(p, st);
    }
    if constexpr (NT > 4 && fit5) {
      if (bsm_env && !p.early_base && lean == 5) return launch_lean<NT, 4, 32, 2, false, true>(p, st);
    }
    constexpr bool fit6 = 2 * NT * 4 * 128 <= 2 * LeanCfg<NT, 4, 16, 2>::STAGE_ELEMS;
    if constexpr (NT > 4 && fit6) {
      if (bsm_env && !p.early_base && lean == 6) return launch_lean<NT, 4, 16, 2, false, true>(p, st);
    }
    switch (lean) {
      case 1: return launch_lean<NT, 4, 16, 4>(p, st);
      case 2: return launch_lean<NT, 4, 32, 3>(p, st);
      case 4: return launch_lean<NT, 4, 16, 3>(p, st);
      case 5: return launch_lean<NT, 4, 32, 2>(p, st);
      case 6: return launch_lean<NT, 4, 16, 2>(p, st);
      default: return launch_lean<NT, 4, 32, 4>(p, st);
    }
  }
  switch (gemm_warps(p.M)) {
    case 8: return launch_cfg<NT, 8>(p, st);
    case 4: return launch_cfg<NT, 4>(p, st);
    default: return launch_cfg<NT, 2>(p, st);
  }
}

bool ts_gemm_ublock_supported(const TsGemmParams& p) {
  // blocks up to 64 wide fuse too (NT 5-8), but measured slower than GEMM + row solves + downdate
  // at config 4 (b = 50: 615 vs ~530 us per iteration; tie at config 5): opt-in, ITERCUR_UB_MAX_N=64
  const int max_n = env_int("ITERCUR_UB_MAX_N", 32);
  return p.N >= 1 && p.N <= std::min(64, max_n) && p.ycp <= 8 * (ts_gemm_nt_host(p.N) + 1) && lean_ok(p) &&
         (p.base_mode == kBaseGatherRowsT || p.base_mode == kBaseGatherCols) &&
         p.norm_part && p.y && p.rt && p.lu && p.yg && p.ctl;
}

int64_t ts_gemm_ublock_parts(int64_t M) { return ceil_div(M, 64); }

template <int NT>
static cudaError_t launch_ublock_nt(const TsGemmParams& p, cudaStream_t st) {
  static const int forced = env_int("ITERCUR_UB_LEAN", env_int("ITERCUR_GEMM_LEAN", -1));
  static const int ub_splits = env_int("ITERCUR_UB_SPLITS", 0);
  // wide blocks need the deeper 32-row stages: the epilogue's LU block and Y(:,J_k) staging
  // (NT = 8: 9.3K doubles + the split-K buffer) must fit the ring
  const int lean = NT > 4 ? 2 : (forced > 0 ? forced : (p.M >= 16000 ? 2 : 1));
  // at most 2 K-splits: only the split-0 CTA runs the (serial) epilogue while its peers wait at
  // the cluster barrier, so deeper splits cost more than they save (config 2, profile-mode
  // phase sums: 7.64 ms at 2 splits vs 7.68 at 3 and 7.99 at 4)
  const int64_t tiles = ceil_div(p.M, 64);
  g_splits_override =
      ub_splits > 0 ? ub_splits : std::min(2, gemm_splits(tiles, p.k_plan > 0 ? p.k_plan : p.K, lean == 2 ? 32 : 16));
  cudaError_t e;
  if constexpr (NT > 4)
    e = launch_lean<NT, 4, 32, 3, true>(p, st);
  else
    e = lean == 2 ? launch_lean<NT, 4, 32, 3, true>(p, st) : launch_lean<NT, 4, 16, 4, true>(p, st);
  g_splits_override = 0;
  return e;
}

// early base loads for blocks up to 32 wide (config 2: 33.2 -> 32.7 ms); wider blocks keep them in
// the epilogue (config 4: no change; config 5, N = 64: 80.3 -> 82 ms, the extra 64 live registers)
static TsGemmParams resolve_early_base(const TsGemmParams& p0) {
  static const int env = env_int("ITERCUR_GEMM_EARLY_BASE", -1);  // A/B: 0 off, 1 on
  TsGemmParams p = p0;
  if (p.early_base < 0) p.early_base = env >= 0 ? env : (p.N <= 32 ? 1 : 0);
  return p;
}

cudaError_t run_ts_gemm_ublock(const TsGemmParams& p0, cudaStream_t st) {
  const TsGemmParams p = resolve_early_base(p0);
  if (!ts_gemm_ublock_supported(p)) return cudaErrorNotSupported;
  if (p.M <= 0) return cudaSuccess;
  switch (ts_gemm_nt_host(p.N)) {
    case 1: return launch_ublock_nt<1>(p, st);
    case 2: return launch_ublock_nt<2>(p, st);
    case 3: return launch_ublock_nt<3>(p, st);
    case 4: return launch_ublock_nt<4>(p, st);
    case 5: return launch_ublock_nt<5>(p, st);
    case 6: return launch_ublock_nt<6>(p, st);
    case 7: return launch_ublock_nt<7>(p, st);
    default: return launch_ublock_nt<8>(p, st);
  }
}

int ts_gemm_nt(int n) { return static_cast<int>(std::min<int64_t>(9, std::max<int64_t>(1, ceil_div(n, 8)))); }

int64_t ts_gemm_grid_size(int64_t M, int N) {
  const int nt = ts_gemm_nt(N);
  return ceil_div(M, gemm_warps(M) * 16) * ceil_div(N, nt * 8);
}

int ts_gemm_planned_splits(const TsGemmParams& p, bool ublock) {
  g_plan_only = true;
  g_planned_z = 0;
  if (ublock)
    run_ts_gemm_ublock(p, nullptr);
  else
    run_ts_gemm(p, nullptr);
  g_plan_only = false;
  return g_planned_z;
}

cudaError_t run_ts_gemm(const TsGemmParams& p0, cudaStream_t st) {
  const TsGemmParams p = resolve_early_base(p0);
  if (p.M <= 0 || p.N <= 0) return cudaSuccess;
  switch (ts_gemm_nt(p.N)) {
    case 1: return launch_nt<1>(p, st);
    case 2: return launch_nt<2>(p, st);
    case 3: return launch_nt<3>(p, st);
    case 4: return launch_nt<4>(p, st);
    case 5: return launch_nt<5>(p, st);
    case 6: return launch_nt<6>(p, st);
    case 7: return launch_nt<7>(p, st);
    case 8: return launch_nt<8>(p, st);
    default: return launch_nt<9>(p, st);
  }
}

// a kernel of this translation unit (module), for itercur_preload
const void* module_anchor_gemm() { return reinterpret_cast<const void*>(ts_gemm_kernel<1, 4>); }

}  // namespace itercur_b200

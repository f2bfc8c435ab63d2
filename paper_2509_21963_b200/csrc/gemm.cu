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

template <int NT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) ts_gemm_kernel(TsGemmParams p) {
  using Cfg = GemmCfg<NT, WARPS>;
  extern __shared__ __align__(16) double gsm[];
  __shared__ double red[WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
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
  const int nk = nvalid > 0 ? static_cast<int>(ceil_div(K, kGemmKT)) : 0;
#pragma unroll
  for (int s = 0; s < kGemmStages - 1; ++s) {
    if (s < nk)
      gemm_load_stage<NT, WARPS>(p, gsm + s * Cfg::STAGE_ELEMS, gsm + s * Cfg::STAGE_ELEMS + Cfg::A_ELEMS, i0,
                                 static_cast<int64_t>(s) * kGemmKT, q0, nvalid, K);
    cp_async_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<kGemmStages - 2>();
    __syncthreads();
    const int nxt = it + kGemmStages - 1;
    if (nxt < nk) {
      double* base = gsm + (nxt % kGemmStages) * Cfg::STAGE_ELEMS;
      gemm_load_stage<NT, WARPS>(p, base, base + Cfg::A_ELEMS, i0, static_cast<int64_t>(nxt) * kGemmKT, q0, nvalid,
                                 K);
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

  // ---------------- epilogue: physical rows (2g, 2g+1), columns (2t, 2t+1) ----------
  double sq = 0.0;
  const int64_t r0 = i0 + warp * 16 + 2 * g;
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
        double base = 0.0;
        switch (p.base_mode) {
          case kBaseGatherCols: base = p.src[i + p.idx[q] * p.lds]; break;
          case kBaseGatherRowsT: base = p.src[p.idx[q] + i * p.lds]; break;
          case kBaseContigCols: base = p.src[i + (p.col0 + q) * p.lds]; break;
          case kBaseInPlaceRowMajor: base = p.C0[i * p.ldc0 + q]; break;
          case kBaseIdentityCols: base = (i == p.col0 + q) ? 1.0 : 0.0; break;
          default: break;
        }
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
}

// CTA height: the largest of {128, 64, 32} rows that still gives >= 4 CTAs per SM.
static int gemm_warps(int64_t M) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("ITERCUR_GEMM_WARPS");  // tuning override: 2, 4 or 8
    forced = e ? atoi(e) : 0;
  }
  if (forced == 2 || forced == 4 || forced == 8) return forced;
  if (ceil_div(M, 128) >= 4 * kNumSMs) return 8;
  if (ceil_div(M, 64) >= 4 * kNumSMs) return 4;
  return 2;
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
  ts_gemm_kernel<NT, WARPS><<<grid, Cfg::THREADS, Cfg::BYTES, st>>>(p);
  return cudaGetLastError();
}

template <int NT>
static cudaError_t launch_nt(const TsGemmParams& p, cudaStream_t st) {
  switch (gemm_warps(p.M)) {
    case 8: return launch_cfg<NT, 8>(p, st);
    case 4: return launch_cfg<NT, 4>(p, st);
    default: return launch_cfg<NT, 2>(p, st);
  }
}

int ts_gemm_nt(int n) { return static_cast<int>(std::min<int64_t>(9, std::max<int64_t>(1, ceil_div(n, 8)))); }

int64_t ts_gemm_grid_size(int64_t M, int N) {
  const int nt = ts_gemm_nt(N);
  return ceil_div(M, gemm_warps(M) * 16) * ceil_div(N, nt * 8);
}

cudaError_t run_ts_gemm(const TsGemmParams& p, cudaStream_t st) {
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

}  // namespace itercur_b200

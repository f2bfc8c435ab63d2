// sketch.cu — the O(mn) stage: Y = S * A applied once over the full matrix
// (proj/src/sketch.cpp:10-24 make_sketch -> proj/src/matrix.cpp:285-289 G*A), with the
// reference's separate ||A||_F zero check (proj/src/driver.cpp:52) fused into the same pass.
//
// Layout: A is column-major m x n (ld lda). The contraction is run as
//     Y^T (n x Np) = A^T (n x m) * S^T (m x Np)
// so the MMA "M" dimension is the columns of A (K = rows of A is contiguous in memory)
// and "N" is the sketch rows padded to a multiple of 8. Tiles of A (16 rows x BM
// columns per TMA box, 128-B swizzle) and of S are staged into shared memory by a
// producer warp with cp.async.bulk.tensor (TMA) through a STAGES-deep mbarrier ring;
// 8 consumer warps run FP64 mma.sync m16n8k8 (DMMA) with K permuted so every fragment
// is one conflict-free 16-byte shared load. ||A||^2 is accumulated from the A fragments
// (each element is loaded exactly once per CTA). Split-K partials are reduced in a fixed
// order by a second kernel, so results are deterministic run to run.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace itercur_b200 {

// ------------------------------------------------------------------ operator generation
// One thread per (h, k) for the Gaussian sketch; one thread per column k of Omega for
// the sparse-sign sketch (partial Fisher-Yates over [0,c), one Philox
// block per slot, sign = low bit of word 1).
__global__ void gen_gaussian_kernel(double* S, int64_t rows_pad, int64_t ldg, int64_t c, int64_t m, uint64_t seed,
                                    uint32_t stream) {
  const int64_t total = rows_pad * ldg;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t h = e / ldg, k = e - h * ldg;
    S[e] = (h < c && k < m) ? normal_at_dev(seed, stream, h, k) : 0.0;
  }
}

__device__ __forceinline__ void sparse_sign_slots(uint64_t seed, int64_t i, int64_t c, int zeta_eff, int32_t* rows,
                                                  int8_t* signs) {
  // partial Fisher-Yates over [0, c): only the <= 2*zeta touched positions are tracked
  int32_t pos[32], val[32];
  int nover = 0;
  auto get = [&](int32_t p) {
    for (int q = 0; q < nover; ++q)
      if (pos[q] == p) return val[q];
    return p;
  };
  auto set = [&](int32_t p, int32_t v) {
    for (int q = 0; q < nover; ++q)
      if (pos[q] == p) { val[q] = v; return; }
    pos[nover] = p;
    val[nover] = v;
    ++nover;
  };
  for (int t = 0; t < zeta_eff; ++t) {
    const U4 r = philox4x32_10(counter_for(kStreamSparseSign, i, t), static_cast<uint32_t>(seed),
                               static_cast<uint32_t>(seed >> 32));
    const uint64_t span = static_cast<uint64_t>(c - t);
    const int32_t jt = t + static_cast<int32_t>((static_cast<uint64_t>(r.x) * span) >> 32);
    const int32_t vt = get(t), vj = get(jt);
    set(t, vj);
    set(jt, vt);
    rows[t] = vj;
    signs[t] = (r.y & 1u) ? -1 : 1;
  }
}

__global__ void gen_sparse_sign_kernel(double* S, int64_t ldg, int64_t c, int64_t m, uint64_t seed, int zeta_eff) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t rows[16];
    int8_t signs[16];
    sparse_sign_slots(seed, k, c, zeta_eff, rows, signs);
    for (int t = 0; t < zeta_eff; ++t) S[rows[t] * ldg + k] = signs[t] > 0 ? 1.0 : -1.0;
  }
}

cudaError_t launch_gen_sketch_operator(double* S, int64_t rows_pad, int64_t ldg, int64_t c, int64_t m, uint64_t seed,
                                       int kind, int zeta, cudaStream_t st, uint32_t stream_tag) {
  if (kind == kSketchGaussian) {
    const int64_t total = rows_pad * ldg;
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 148 * 16));
    gen_gaussian_kernel<<<blocks, 256, 0, st>>>(S, rows_pad, ldg, c, m, seed, stream_tag);
  } else {
    cudaError_t e = cudaMemsetAsync(S, 0, sizeof(double) * rows_pad * ldg, st);
    if (e != cudaSuccess) return e;
    const int ze = static_cast<int>(std::min<int64_t>(zeta, c));
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(m, 256), 148 * 16));
    gen_sparse_sign_kernel<<<blocks, 256, 0, st>>>(S, ldg, c, m, seed, ze);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ DMMA sketch kernel
constexpr int kWarps = 8;        // consumer warps
constexpr int kThreads = (kWarps + 1) * 32;

template <int NT, int MT, int KS>
struct SketchCfg {
  static constexpr int BM = kWarps * MT * 16;  // columns of A per CTA
  static constexpr int N = NT * 8;             // sketch rows handled per CTA
  static constexpr int SUB = KS / 16;          // 16-row TMA boxes per stage
  static constexpr int A_SUB_BYTES = BM * 128;
  static constexpr int G_SUB_BYTES = N * 128;
  static constexpr int STAGE_BYTES = SUB * (A_SUB_BYTES + G_SUB_BYTES);
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES >= 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int NT, int MT, int KS>
__device__ __forceinline__ void compute_stage(const char* sA, const char* sG, double (&acc)[MT][NT][4], double& asq,
                                              int warp, int lane) {
  using Cfg = SketchCfg<NT, MT, KS>;
  const uint32_t g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int sub = 0; sub < Cfg::SUB; ++sub) {
    const char* a_sub = sA + sub * Cfg::A_SUB_BYTES;
    const char* g_sub = sG + sub * Cfg::G_SUB_BYTES;
#pragma unroll
    for (int kk = 0; kk < 16; kk += 8) {
      double2 af[MT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const uint32_t row0 = (warp * MT + mt) * 16 + g;
        af[mt][0] = *reinterpret_cast<const double2*>(a_sub + sw128_offset(row0, kk + 2 * t));
        af[mt][1] = *reinterpret_cast<const double2*>(a_sub + sw128_offset(row0 + 8, kk + 2 * t));
        asq = fma(af[mt][0].x, af[mt][0].x, asq);
        asq = fma(af[mt][0].y, af[mt][0].y, asq);
        asq = fma(af[mt][1].x, af[mt][1].x, asq);
        asq = fma(af[mt][1].y, af[mt][1].y, asq);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const double2 bf = *reinterpret_cast<const double2*>(g_sub + sw128_offset(nt * 8 + g, kk + 2 * t));
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          dmma_16x8x8(acc[mt][nt], af[mt][0].x, af[mt][1].x, af[mt][0].y, af[mt][1].y, bf.x, bf.y);
      }
    }
  }
}

// grid: x = column tiles (BM), y = K splits, z = N chunks (each NT*8 sketch rows)
template <int NT, int MT, int KS, bool TMA>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmG,
                       const double* __restrict__ A, int64_t lda, const double* __restrict__ S, int64_t ldg,
                       int64_t m, int64_t n, int64_t Np, int64_t k_per_split, double* __restrict__ Yout,
                       int64_t split_stride, double* __restrict__ asq_part) {
  using Cfg = SketchCfg<NT, MT, KS>;
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  __shared__ double red[kWarps + 1];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * Cfg::BM;
  const int64_t k_begin = static_cast<int64_t>(blockIdx.y) * k_per_split;
  const int64_t k_end = min(m, k_begin + k_per_split);
  const int64_t n_off = static_cast<int64_t>(blockIdx.z) * Cfg::N;
  const int nk = static_cast<int>(k_end > k_begin ? ceil_div(k_end - k_begin, KS) : 0);

  auto stageA = [&](int s, int sub) { return smem + s * Cfg::STAGE_BYTES + sub * Cfg::A_SUB_BYTES; };
  auto stageG = [&](int s, int sub) {
    return smem + s * Cfg::STAGE_BYTES + Cfg::SUB * Cfg::A_SUB_BYTES + sub * Cfg::G_SUB_BYTES;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TMA ? kWarps : kThreads);
    }
    fence_barrier_init();
  }
  __syncthreads();

  double acc[MT][NT][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[mt][nt][v] = 0.0;
  double asq = 0.0;

  if constexpr (TMA) {
    if (warp == kWarps) {
      // ---------------- producer warp: one elected lane drives the TMA ring ----------
      if (lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmG);
        for (int it = 0; it < nk; ++it) {
          const int s = it % Cfg::STAGES;
          const uint32_t phase = (it / Cfg::STAGES) & 1u;
          mbar_wait(&empty[s], phase ^ 1u);
          mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
          const int32_t kc = static_cast<int32_t>(k_begin + static_cast<int64_t>(it) * KS);
#pragma unroll
          for (int sub = 0; sub < Cfg::SUB; ++sub) {
            tma_load_2d(stageA(s, sub), &tmA, &full[s], kc + sub * 16, static_cast<int32_t>(j0));
            tma_load_2d(stageG(s, sub), &tmG, &full[s], kc + sub * 16, static_cast<int32_t>(n_off));
          }
        }
      }
      __syncwarp();
    } else {
      // ---------------- consumer warps ------------------------------------------------
      for (int it = 0; it < nk; ++it) {
        const int s = it % Cfg::STAGES;
        const uint32_t phase = (it / Cfg::STAGES) & 1u;
        mbar_wait(&full[s], phase);
        compute_stage<NT, MT, KS>(stageA(s, 0), stageG(s, 0), acc, asq, warp, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
      }
    }
  } else {
    // ------------- fallback (A not TMA-compatible, e.g. odd lda): all threads stage ---
    for (int it = 0; it < nk; ++it) {
      const int64_t kc = k_begin + static_cast<int64_t>(it) * KS;
      char* sa = stageA(0, 0);
      char* sg = stageG(0, 0);
      for (int e = threadIdx.x; e < Cfg::BM * KS; e += kThreads) {
        const int jl = e / KS, kl = e % KS;
        const int64_t k = kc + kl, j = j0 + jl;
        const double v = (k < m && j < n) ? A[k + j * lda] : 0.0;
        *reinterpret_cast<double*>(sa + (kl / 16) * Cfg::A_SUB_BYTES + sw128_offset(jl, kl % 16)) = v;
      }
      for (int e = threadIdx.x; e < Cfg::N * KS; e += kThreads) {
        const int hl = e / KS, kl = e % KS;
        const int64_t k = kc + kl, h = n_off + hl;
        const double v = (k < m && h < Np) ? S[h * ldg + k] : 0.0;
        *reinterpret_cast<double*>(sg + (kl / 16) * Cfg::G_SUB_BYTES + sw128_offset(hl, kl % 16)) = v;
      }
      __syncthreads();
      if (warp < kWarps) compute_stage<NT, MT, KS>(sa, sg, acc, asq, warp, lane);
      __syncthreads();
    }
  }

  // ---------------- epilogue: Y^T tile rows j, sketch rows h (16-byte stores) ----------
  if (warp < kWarps) {
    const int g = lane >> 2, t = lane & 3;
    double* out = Yout + static_cast<int64_t>(blockIdx.y) * split_stride;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int64_t j = j0 + (warp * MT + mt) * 16 + g + 8 * half;
        if (j < n) {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int64_t h = n_off + nt * 8 + 2 * t;
            if (h < Np)
              *reinterpret_cast<double2*>(out + j * Np + h) =
                  make_double2(acc[mt][nt][2 * half], acc[mt][nt][2 * half + 1]);
          }
        }
      }
    }
  }
  // ||A||^2 partial: only the z == 0 slice owns it (every slice re-reads the same A).
  double v = warp < kWarps ? warp_sum(asq) : 0.0;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tsum = 0.0;
    for (int w = 0; w < kWarps; ++w) tsum += red[w];
    if (blockIdx.z == 0) asq_part[blockIdx.y * gridDim.x + blockIdx.x] = tsum;
  }
}

// Fixed-order split reduction + scale + ||Y||^2 block partials.
__global__ void sketch_reduce_kernel(const double* __restrict__ part, int splits, int64_t split_stride,
                                     double scale, double* __restrict__ Y, int64_t total, double* __restrict__ ysq_part) {
  __shared__ double red[8];
  double sq = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < splits; ++p) s += part[p * split_stride + e];
    s *= scale;
    Y[e] = s;
    sq = fma(s, s, sq);
  }
  const double b = block_sum<256>(sq, red);
  if (threadIdx.x == 0) ysq_part[blockIdx.x] = b;
}

// Sum `count` partials in index order into *out (single block; deterministic).
__global__ void reduce_partials_kernel(const double* __restrict__ p, int count, double* __restrict__ out) {
  __shared__ double red[8];
  // strided accumulation per thread, then fixed tree: deterministic for fixed count
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += p[i];
  const double b = block_sum<256>(s, red);
  if (threadIdx.x == 0) *out = b;
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static bool make_tmap_2d(CUtensorMap* map, const double* base, uint64_t dim0, uint64_t dim1, uint64_t ld_elems,
                         uint32_t box0, uint32_t box1) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15u) != 0 || (ld_elems * 8) % 16 != 0) return false;
  if (dim0 >= (1ull << 32) || dim1 >= (1ull << 32)) return false;
  cuuint64_t dims[2] = {dim0, dim1};
  cuuint64_t strides[1] = {ld_elems * 8};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

using SketchKernelFn = void (*)(CUtensorMap, CUtensorMap, const double*, int64_t, const double*, int64_t, int64_t,
                                int64_t, int64_t, int64_t, double*, int64_t, double*);

template <int NT, int MT = 1, int KS = 32>
static SketchKernelFn pick_kernel(bool tma, int* smem_bytes, int* bm) {
  // Only the validated tile shape is instantiated: the round-1 two-m-tile / 16-row-stage variant
  // (MT = 2, KS = 16) produced runaway ranks at config 3 and was never root-caused, so it is not
  // buildable (bitwise determinism at config 3's shape: tests/test_gpu_stages.py).
  static_assert(MT == 1 && KS == 32, "sketch_dmma_kernel: only MT = 1, KS = 32 is validated");
  using Cfg = SketchCfg<NT, MT, KS>;
  *smem_bytes = Cfg::SMEM_BYTES;
  *bm = Cfg::BM;
  if (tma) return sketch_dmma_kernel<NT, MT, KS, true>;
  return sketch_dmma_kernel<NT, MT, KS, false>;
}

static SketchKernelFn kernel_for_nt(int nt, bool tma, int* smem, int* bm) {
  switch (nt) {
    case 1: return pick_kernel<1>(tma, smem, bm);
    case 2: return pick_kernel<2>(tma, smem, bm);
    case 3: return pick_kernel<3>(tma, smem, bm);
    case 4: return pick_kernel<4>(tma, smem, bm);
    case 5: return pick_kernel<5>(tma, smem, bm);
    case 6: return pick_kernel<6>(tma, smem, bm);
    case 7: return pick_kernel<7>(tma, smem, bm);
    case 8: return pick_kernel<8>(tma, smem, bm);
    default: return pick_kernel<9>(tma, smem, bm);
  }
}

struct SketchPlan {
  int nt, nchunks, bm, smem, splits, col_tiles;
  int64_t kps;
  bool tma;
};

static SketchPlan plan_sketch(int64_t m, int64_t n, int64_t lda, const double* A, int64_t c_pad) {
  SketchPlan p{};
  const int ntiles_total = static_cast<int>(c_pad / 8);
  p.nchunks = static_cast<int>(ceil_div(ntiles_total, 9));
  p.nt = static_cast<int>(ceil_div(ntiles_total, p.nchunks));
  p.tma = ((reinterpret_cast<uintptr_t>(A) & 15u) == 0) && ((lda * 8) % 16 == 0) && get_encode_fn() != nullptr &&
          m < (1ll << 31) && n < (1ll << 31);
  kernel_for_nt(p.nt, p.tma, &p.smem, &p.bm);
  p.col_tiles = static_cast<int>(ceil_div(n, p.bm));
  // choose K splits so the grid fills whole waves of 148 SMs (1 CTA / SM)
  const int64_t ktiles = ceil_div(m, 32);
  int best_s = 1;
  double best_score = -1.0;
  for (int s = 1; s <= 64 && s <= ktiles; ++s) {
    const int64_t ctas = static_cast<int64_t>(p.col_tiles) * s * p.nchunks;
    const double waves = static_cast<double>(ctas) / kNumSMs;
    const double eff = waves / std::ceil(waves);
    const double per_cta_k = static_cast<double>(ktiles) / s;
    // penalise tiny K per CTA (pipeline fill) and partial traffic
    const double score = eff - (per_cta_k < 8 ? 0.2 : 0.0) - 0.004 * s;
    if (score > best_score + 1e-9) { best_score = score; best_s = s; }
  }
  p.splits = best_s;
  p.kps = ceil_div(ktiles, best_s) * 32;
  p.splits = static_cast<int>(ceil_div(m, p.kps));
  return p;
}

int64_t sketch_workspace_elems(int64_t m, int64_t n, int64_t c_pad) {
  SketchPlan p = plan_sketch(m, n, m + (m & 1), reinterpret_cast<const double*>(uintptr_t(256)), c_pad);
  // partial Y per split (only when splits > 1) + asq partials + ysq partials
  return (p.splits > 1 ? static_cast<int64_t>(p.splits) * n * c_pad : 0) +
         static_cast<int64_t>(p.col_tiles) * p.splits + 4096;
}

static cudaError_t launch_dmma(const SketchPlan& p, const double* A, int64_t m, int64_t n, int64_t lda,
                               const double* S, int64_t ldg, int64_t c_pad, double* out, int64_t split_stride,
                               double* asq_part, cudaStream_t st) {
  int smem = 0, bm = 0;
  SketchKernelFn fn = kernel_for_nt(p.nt, p.tma, &smem, &bm);
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  CUtensorMap tmA{}, tmG{};
  if (p.tma) {
    if (!make_tmap_2d(&tmA, A, m, n, lda, 16, bm)) return cudaErrorInvalidValue;
    if (!make_tmap_2d(&tmG, S, ldg, c_pad, ldg, 16, p.nt * 8)) return cudaErrorInvalidValue;
  }
  dim3 grid(p.col_tiles, p.splits, p.nchunks);
  fn<<<grid, kThreads, smem, st>>>(tmA, tmG, A, lda, S, ldg, m, n, c_pad, p.kps, out, split_stride, asq_part);
  return cudaGetLastError();
}

cudaError_t run_sketch_apply(const double* A, int64_t m, int64_t n, int64_t lda, const double* S, int64_t ldg,
                             int64_t c_pad, double scale, double* Y, double* ws, int64_t ws_elems,
                             const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info) {
  SketchPlan p = plan_sketch(m, n, lda, A, c_pad);
  const int64_t part_elems = p.splits > 1 ? static_cast<int64_t>(p.splits) * n * c_pad : 0;
  const int64_t asq_count = static_cast<int64_t>(p.col_tiles) * p.splits;
  if (part_elems + asq_count + 4096 > ws_elems) return cudaErrorInvalidValue;
  double* part = ws;
  double* asq_part = ws + part_elems;
  double* ysq_part = asq_part + asq_count;
  double* out = p.splits > 1 ? part : Y;
  cudaError_t e = launch_dmma(p, A, m, n, lda, S, ldg, c_pad, out, n * c_pad, asq_part, st);
  if (e != cudaSuccess) return e;
  const int64_t total = n * c_pad;
  const int rblocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 2048));
  sketch_reduce_kernel<<<rblocks, 256, 0, st>>>(part_elems ? part : Y, p.splits > 1 ? p.splits : 1, n * c_pad,
                                                scale, Y, total, ysq_part);
  reduce_partials_kernel<<<1, 256, 0, st>>>(ysq_part, rblocks, stats.d_ysq);
  reduce_partials_kernel<<<1, 256, 0, st>>>(asq_part, static_cast<int>(asq_count), stats.d_asq);
  if (info) {
    info->splits = p.splits;
    info->ctas = p.col_tiles * p.splits * p.nchunks;
    info->nt = p.nt;
    info->tma = p.tma;
    info->dominant_launches = 1;
  }
  return cudaGetLastError();
}

cudaError_t run_sketch_dmma_only(const double* A, int64_t m, int64_t n, int64_t lda, const double* S, int64_t ldg,
                                 int64_t c_pad, double* Y, double* ws, int64_t ws_elems, cudaStream_t st,
                                 SketchLaunchInfo* info) {
  SketchPlan p = plan_sketch(m, n, lda, A, c_pad);
  const int64_t part_elems = p.splits > 1 ? static_cast<int64_t>(p.splits) * n * c_pad : 0;
  const int64_t asq_count = static_cast<int64_t>(p.col_tiles) * p.splits;
  if (part_elems + asq_count + 4096 > ws_elems) return cudaErrorInvalidValue;
  double* out = p.splits > 1 ? ws : Y;
  if (info) {
    info->splits = p.splits;
    info->ctas = p.col_tiles * p.splits * p.nchunks;
    info->nt = p.nt;
    info->tma = p.tma;
    info->dominant_launches = 1;
  }
  return launch_dmma(p, A, m, n, lda, S, ldg, c_pad, out, n * c_pad, ws + part_elems, st);
}


// ------------------------------------------------------------------ sparse-sign sketch
// Y = Omega * A with Omega's zeta nonzeros (+-1) per column applied as a
// sparse operator: 8 adds per element of A instead of 2 * c_pad DMMA flops. A is streamed
// once in 256-row x 32-column tiles (coalesced 8-byte loads, register-prefetched one tile
// ahead, staged in shared memory with an odd pitch); the operator is kept transposed per
// 256-row tile: for each sketch row h, the tile rows it touches in ascending order with
// their signs (16-bit entries). Warp q owns sketch rows h = q, q + 16, ..; lane j owns
// column j of the tile, so every list entry is one broadcast 16-bit load plus one
// conflict-free 256-byte row read per warp. Each Y(h, j) is a running sum over ascending
// rows i from 0 with the sign applied as add / subtract, then scaled once: the same
// operations in the same order as the oracle's sparse loop (bitwise-identical Y).
constexpr int kSpTI = 256;   // rows per tile
constexpr int kSpTJ = 32;    // columns per CTA
constexpr int kSpThreads = 512;
constexpr int kSpMaxC = 128;  // sketch rows supported (8 accumulators per lane)
// per-tile list capacity: zeta entries per row plus up to 3 padding entries per sketch row
__host__ __device__ constexpr int sp_list_cap(int zeta, int c_pad) { return zeta * kSpTI + 4 * c_pad; }

constexpr int kSpTJP = kSpTJ + 1;  // odd tile pitch: a lane-per-row store hits distinct bank pairs
// lists of tile t: entries[t * zeta * 256 + off[t * (c_pad + 1) + h] ...]; an entry is the row's
// byte offset in the tile (row * kSpTJP * 8) with the sign in bit 31 (xor into the value's sign)
__global__ void __launch_bounds__(kSpTI) sparse_lists_kernel(uint64_t seed, int64_t m, int c, int c_pad, int zeta,
                                                             uint32_t* __restrict__ entries, int* __restrict__ offs) {
  __shared__ int cnt[kSpTI / 32][kSpMaxC];
  __shared__ int base[kSpTI / 32][kSpMaxC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kSpTI + threadIdx.x;
  int32_t rows[16];
  int8_t signs[16];
  uint32_t hit[kSpMaxC / 32] = {0, 0, 0, 0}, neg[kSpMaxC / 32] = {0, 0, 0, 0};
  if (i < m) {
    sparse_sign_slots(seed, i, c, zeta, rows, signs);
    for (int t = 0; t < zeta; ++t) {
      hit[rows[t] >> 5] |= 1u << (rows[t] & 31);
      if (signs[t] < 0) neg[rows[t] >> 5] |= 1u << (rows[t] & 31);
    }
  }
  for (int h = 0; h < c; ++h) {
    const unsigned bal = __ballot_sync(0xffffffffu, hit[h >> 5] >> (h & 31) & 1u);
    if (lane == 0) cnt[warp][h] = __popc(bal);
  }
  __syncthreads();
  __shared__ int pad_from[kSpMaxC], pad_to[kSpMaxC];
  if (threadIdx.x == 0) {
    int run = 0;
    int* o = offs + static_cast<int64_t>(blockIdx.x) * (c_pad + 1);
    for (int h = 0; h < c_pad; ++h) {
      o[h] = run;
      for (int w = 0; w < kSpTI / 32; ++w) {
        base[w][h] = run;
        run += h < c ? cnt[w][h] : 0;
      }
      pad_from[h] = run;
      run = (run + 3) & ~3;  // every list a multiple of 4 entries
      pad_to[h] = run;
    }
    o[c_pad] = run;
  }
  __syncthreads();
  uint32_t* e = entries + static_cast<int64_t>(blockIdx.x) * sp_list_cap(zeta, c_pad);
  for (int h = threadIdx.x; h < c_pad; h += kSpTI)
    for (int q = pad_from[h]; q < pad_to[h]; ++q) e[q] = static_cast<uint32_t>(kSpTI * kSpTJP * 8);  // zero row
  for (int h = 0; h < c; ++h) {
    const bool mine = hit[h >> 5] >> (h & 31) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, mine);
    if (mine) {
      const int pos = base[warp][h] + __popc(bal & ((1u << lane) - 1u));
      e[pos] = static_cast<uint32_t>(threadIdx.x * kSpTJP * 8) | ((neg[h >> 5] >> (h & 31) & 1u) << 31);
    }
  }
}

template <int NH>  // accumulators per lane: sketch rows q, q + 16, .. (NH * 16 >= c_pad)
__global__ void __launch_bounds__(kSpThreads, 1)
    sparse_sketch_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                         const uint32_t* __restrict__ entries, const int* __restrict__ offs, int c, int c_pad,
                         int zeta, double scale, double* __restrict__ Y, double* __restrict__ asq_part,
                         double* __restrict__ ysq_part, int mode) {
  constexpr int TJP = kSpTJP;
  extern __shared__ __align__(16) double sps[];
  double* tile = sps;                                                    // [kSpTI + 1][TJP], last row 0
  uint32_t* lst = reinterpret_cast<uint32_t*>(tile + (kSpTI + 1) * TJP + 1);  // [list cap], 16-byte aligned
  int* off = reinterpret_cast<int*>(lst + sp_list_cap(16, kSpMaxC));     // [c_pad + 1]
  __shared__ double red[kSpThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kSpTJ;
  const int ntiles = static_cast<int>((m + kSpTI - 1) / kSpTI);
  // loader: warp w reads columns w and w + 16, lane l rows l + 32u of the tile
  const int64_t jl0 = j0 + warp, jl1 = j0 + warp + 16;
  const bool c0ok = jl0 < n, c1ok = jl1 < n;
  const double* a0 = A + (c0ok ? jl0 : 0) * lda;
  const double* a1 = A + (c1ok ? jl1 : 0) * lda;
  double pre[16];
  constexpr int kLpre = (sp_list_cap(16, kSpMaxC) / 4 + kSpThreads - 1) / kSpThreads;
  uint4 lpre[kLpre];  // this tile's operator lists
  int opre = 0;       // and one list offset
  const int nent4 = sp_list_cap(zeta, c_pad) / 4;
  if (threadIdx.x < TJP) tile[kSpTI * TJP + threadIdx.x] = 0.0;  // the zero row (padding entries)
  double asq = 0.0;
  auto fetch = [&](int t) {
    const int64_t i0 = static_cast<int64_t>(t) * kSpTI;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + lane + 32 * u;
      pre[u] = (c0ok && i < m) ? __ldcs(a0 + i) : 0.0;
      pre[8 + u] = (c1ok && i < m) ? __ldcs(a1 + i) : 0.0;
    }
    const uint4* src = reinterpret_cast<const uint4*>(entries) + static_cast<int64_t>(t) * nent4;
#pragma unroll
    for (int k = 0; k < kLpre; ++k) {
      const int q = threadIdx.x + k * kSpThreads;
      lpre[k] = q < nent4 ? src[q] : make_uint4(0, 0, 0, 0);
    }
    opre = threadIdx.x <= c_pad ? offs[static_cast<int64_t>(t) * (c_pad + 1) + threadIdx.x] : 0;
  };
  double acc[NH];
#pragma unroll
  for (int q = 0; q < NH; ++q) acc[q] = 0.0;
  fetch(0);
  for (int t = 0; t < ntiles; ++t) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      tile[(lane + 32 * u) * TJP + warp] = pre[u];
      tile[(lane + 32 * u) * TJP + warp + 16] = pre[8 + u];
      asq = fma(pre[u], pre[u], asq);
      asq = fma(pre[8 + u], pre[8 + u], asq);
    }
#pragma unroll
    for (int k = 0; k < kLpre; ++k) {
      const int q = threadIdx.x + k * kSpThreads;
      if (q < nent4) reinterpret_cast<uint4*>(lst)[q] = lpre[k];
    }
    if (threadIdx.x <= c_pad) off[threadIdx.x] = opre;
    __syncthreads();
    if (t + 1 < ntiles && !(mode & 2)) fetch(t + 1);  // next tile in flight during the list walk
    const uint32_t col = smem_u32(tile) + lane * 8;
    auto add_entry = [&](double v, uint32_t u) {
      // v + (x with its sign flipped when u's bit 31 is set) == v -/+ x exactly
      double x;
      asm("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(col + (u & 0x7fffffffu)));  // (not volatile: the 4 loads batch)
      const int hi = __double2hiint(x) ^ static_cast<int>(u & 0x80000000u);
      return __dadd_rn(v, __hiloint2double(hi, __double2loint(x)));
    };
    // Every list is padded to a multiple of 4 entries that read the tile's zero row (adding
    // +0.0 leaves a running sum that started at +0.0 unchanged, so Y stays bitwise the oracle's),
    // so 4 entries arrive per broadcast 16-byte load: one shared-memory wavefront per 4.
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const int h = warp + 16 * q;
      if (h >= c || (mode & 1)) continue;
      const int e0 = off[h], e1 = off[h + 1];
      double v = acc[q];
      for (int e = e0; e < e1; e += 8) {
        const uint4 ua = *reinterpret_cast<const uint4*>(lst + e);
        const uint4 ub = e + 4 < e1 ? *reinterpret_cast<const uint4*>(lst + e + 4) : make_uint4(0, 0, 0, 0);
        v = add_entry(v, ua.x);
        v = add_entry(v, ua.y);
        v = add_entry(v, ua.z);
        v = add_entry(v, ua.w);
        if (e + 4 < e1) {
          v = add_entry(v, ub.x);
          v = add_entry(v, ub.y);
          v = add_entry(v, ub.z);
          v = add_entry(v, ub.w);
        }
      }
      acc[q] = v;
    }
    __syncthreads();
  }
  double ysq = 0.0;
  const int64_t j = j0 + lane;
#pragma unroll
  for (int q = 0; q < NH; ++q) {
    const int h = warp + 16 * q;
    if (h < c_pad && j < n) {
      const double v = h < c ? acc[q] * scale : 0.0;
      Y[h + j * c_pad] = v;
      ysq = fma(v, v, ysq);
    }
  }
  const double bs = block_sum<kSpThreads>(asq, red);
  if (threadIdx.x == 0) asq_part[blockIdx.x] = bs;
  __syncthreads();
  const double by = block_sum<kSpThreads>(ysq, red);
  if (threadIdx.x == 0) ysq_part[blockIdx.x] = by;
}

int64_t sparse_sketch_workspace_elems(int64_t m, int64_t n, int64_t c_pad, int zeta) {
  const int64_t tiles = ceil_div(m, kSpTI);
  const int64_t ent_bytes = tiles * sp_list_cap(zeta, static_cast<int>(c_pad)) * 4, off_bytes = tiles * (c_pad + 1) * 4;
  return ceil_div(ent_bytes + off_bytes, 8) + 2 * ceil_div(n, kSpTJ) + 16;
}

bool sparse_sketch_supported(int64_t c, int zeta) { return c >= 1 && c <= kSpMaxC && zeta >= 1 && zeta <= 16; }

cudaError_t run_sketch_apply_sparse(const double* A, int64_t m, int64_t n, int64_t lda, uint64_t seed, int64_t c,
                                    int64_t c_pad, int zeta, double scale, double* Y, double* ws, int64_t ws_elems,
                                    const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info) {
  if (!sparse_sketch_supported(c, zeta) || c_pad > kSpMaxC) return cudaErrorInvalidValue;
  if (sparse_sketch_workspace_elems(m, n, c_pad, zeta) > ws_elems) return cudaErrorInvalidValue;
  const int64_t tiles = ceil_div(m, kSpTI), ctas = ceil_div(n, kSpTJ);
  uint32_t* entries = reinterpret_cast<uint32_t*>(ws);
  const int64_t cap = sp_list_cap(zeta, static_cast<int>(c_pad));
  int* offs = reinterpret_cast<int*>(entries + tiles * cap);
  double* asq_part = ws + ceil_div(tiles * cap * 4 + tiles * (c_pad + 1) * 4, 8);
  double* ysq_part = asq_part + ctas;
  sparse_lists_kernel<<<static_cast<unsigned>(tiles), kSpTI, 0, st>>>(seed, m, static_cast<int>(c),
                                                                     static_cast<int>(c_pad), zeta, entries, offs);
  const size_t smem = sizeof(double) * ((kSpTI + 1) * kSpTJP + 1) + 4 * sp_list_cap(16, kSpMaxC) + 4 * (kSpMaxC + 1);
  auto launch = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    static const int mode = getenv("ITERCUR_SPARSE_MODE") ? atoi(getenv("ITERCUR_SPARSE_MODE")) : 0;  // ablation
    kern<<<static_cast<unsigned>(ctas), kSpThreads, smem, st>>>(A, m, n, lda, entries, offs, static_cast<int>(c),
                                                                static_cast<int>(c_pad), zeta, scale, Y, asq_part,
                                                                ysq_part, mode);
    return cudaGetLastError();
  };
  cudaError_t e;
  if (c_pad <= 16) e = launch(sparse_sketch_kernel<1>);
  else if (c_pad <= 32) e = launch(sparse_sketch_kernel<2>);
  else if (c_pad <= 64) e = launch(sparse_sketch_kernel<4>);
  else e = launch(sparse_sketch_kernel<8>);
  if (e != cudaSuccess) return e;
  reduce_partials_kernel<<<1, 256, 0, st>>>(ysq_part, static_cast<int>(ctas), stats.d_ysq);
  reduce_partials_kernel<<<1, 256, 0, st>>>(asq_part, static_cast<int>(ctas), stats.d_asq);
  if (info) {
    info->splits = 1;
    info->ctas = static_cast<int>(ctas);
    info->nt = 0;
    info->tma = false;
    info->dominant_launches = 1;
  }
  return cudaGetLastError();
}


// ------------------------------------------------------------------ sparse-sign sketch, sliced-integer form
// Y = Omega * A for the sparse-sign operator (+-1 at zeta positions per column of Omega, SURVEY.md
// A.8; the scale 1/sqrt(zeta) is applied once by the reduce). The +-1 entries are exact in int8,
// so the contraction runs on the integer tensor path (mma.sync m16n8k32 s8 x u8/s8 -> s32,
// measured 1.1 POP/s on B200, tools/microbench/sparse_dispatch.cu) instead of FP64 DMMA: every
// element x of A is written as a 56-bit two's-complement fixed-point integer relative to a
// running per-column exponent E (the largest exponent seen so far in that column of this CTA's
// row range): w = rint(x * 2^(1076 - E)), |w| < 2^54, and its 7 bytes are 7 int8 slices
// (bytes 0..5 unsigned, byte 6 signed). Each slice is one MMA with the int8 operator tile; the
// int32 accumulators are exact and are folded into FP64 (sum_t 2^(8t) acc_t * 2^(E - 1076))
// only when a column's exponent grows (rare: once or twice per column) and at the end. The
// per-element representation error is <= 2^(E-1077) (half an ulp of a 54-bit mantissa at the
// column's running maximum), i.e. below FP64's own rounding of the sums.
// Why: at c_pad = 56 (config 4) the DMMA form needs 112 flop per 8-byte element, 2.4x past the
// FP64 ridge (37 TF / 6.45 TB/s); the sliced form needs 7 x 128 integer ops per element at
// 1.1 POP/s, which sits under the HBM time.
// Tiling: CTA = 4 warps x 8 columns (32 columns of A), K in steps of 32 rows staged by cp.async
// through a cp.async ring (im_stages) (A tile: 32 columns x 256 B, column pitch 272 B: conflict-free 16-byte
// fragment loads; operator tile: 16*MT rows x 32 B, pitch 48 B: conflict-free ldmatrix).
// Warp fragment: A operand = operator tile (16*MT sketch rows x 32 rows of A, row-major, ldmatrix
// .x4 per 16 sketch rows), B operand = slices of 32 rows x 8 columns (thread: column lane/4,
// rows 4(lane%4)+{0..3} and +16: two 32-byte runs of its column), C = 16 sketch rows x 8 columns.
constexpr int kImWarps = 4;
constexpr int kImThreads = kImWarps * 32;
constexpr int kImCols = kImWarps * 8;   // columns of A per CTA
constexpr int kImColPitch = 272;        // bytes per staged column (32 doubles + 16)
constexpr int kImOmPitch = 48;          // bytes per staged operator row (32 + 16)
// ring depth: 2 CTAs per SM at MT >= 3 (registers), 3 below; deep enough for ~110 KB of A in
// flight per SM either way
template <int MT>
constexpr int im_stages() { return MT <= 2 ? 6 : 8; }
constexpr int kImSlices = 7;

template <int MT>
struct ImCfg {
  static constexpr int kAStage = kImCols * kImColPitch;       // 8704 B
  static constexpr int kOStage = 16 * MT * kImOmPitch;        // 768 * MT B
  static constexpr int kStage = kAStage + kOStage;
  static constexpr int kYacc = kImWarps * 16 * MT * 8 * 8;    // fp64 accumulators per warp: 16*MT x 8
  static constexpr int kStages = im_stages<MT>();
  static constexpr int kSmem = kStages * kStage + kYacc;
};

__global__ void gen_sparse_sign_i8_kernel(int8_t* O, int64_t ld8, int64_t c, int64_t m, uint64_t seed, int zeta_eff) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t rows[16];
    int8_t signs[16];
    sparse_sign_slots(seed, k, c, zeta_eff, rows, signs);
    for (int t = 0; t < zeta_eff; ++t) O[rows[t] * ld8 + k] = signs[t];
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <bool SIGNED_B>
__device__ __forceinline__ void imma_16x8x32(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (SIGNED_B)
    asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 2^e for e in [-1022, 1023] (exact)
__device__ __forceinline__ double pow2i(int e) { return __hiloint2double((e + 1023) << 20, 0); }

// bytes t of four 64-bit integers (lo words l0..l3, hi words h0..h3) -> slice registers s[0..6]
__device__ __forceinline__ void byte_transpose(uint32_t l0, uint32_t l1, uint32_t l2, uint32_t l3, uint32_t h0,
                                               uint32_t h1, uint32_t h2, uint32_t h3, uint32_t (&s)[kImSlices]) {
  const uint32_t a = __byte_perm(l0, l1, 0x5140), b = __byte_perm(l2, l3, 0x5140);
  const uint32_t c = __byte_perm(l0, l1, 0x7362), d = __byte_perm(l2, l3, 0x7362);
  s[0] = __byte_perm(a, b, 0x5410);
  s[1] = __byte_perm(a, b, 0x7632);
  s[2] = __byte_perm(c, d, 0x5410);
  s[3] = __byte_perm(c, d, 0x7632);
  const uint32_t e = __byte_perm(h0, h1, 0x5140), f = __byte_perm(h2, h3, 0x5140);
  const uint32_t g = __byte_perm(h0, h1, 0x7362), h = __byte_perm(h2, h3, 0x7362);
  s[4] = __byte_perm(e, f, 0x5410);
  s[5] = __byte_perm(e, f, 0x7632);
  s[6] = __byte_perm(g, h, 0x5410);
}

template <int MT, int NS>  // NS slices: bytes 0..NS-1 of w = rint(x * 2^(kSh - E)), top byte signed
__global__ void __launch_bounds__(kImThreads, (MT <= 2 ? 3 : 2))
    sparse_sketch_imma_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                              const int8_t* __restrict__ O, int64_t ld8, int64_t kps, int64_t c_pad,
                              double* __restrict__ part, int64_t split_stride, double* __restrict__ asq_part) {
  using Cfg = ImCfg<MT>;
  constexpr int kSh = 1076 - 8 * (7 - NS);  // |w| < 2^(8 NS - 3)
  extern __shared__ __align__(128) uint8_t ims[];
  double* yacc = reinterpret_cast<double*>(ims + Cfg::kStages * Cfg::kStage);
  __shared__ double red[kImWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kImCols;
  const int64_t kb = static_cast<int64_t>(blockIdx.y) * kps * 32;
  const int64_t ke = m < kb + kps * 32 ? m : kb + kps * 32;
  const int nsteps = static_cast<int>(ke > kb ? (ke - kb + 31) / 32 : 0);
  const uint32_t sbase = smem_u32(ims);

  // producer mapping: A tile = 32 columns x 16 chunks of 16 B (thread: chunk tid & 15 of columns
  // tid / 16 + 8u, u = 0..3); operator tile = 16*MT rows x 2 chunks (threads < 32*MT). Per-thread
  // source pointers advance by one k-step (32 rows) per stage; only the last k-steps of the CTA's
  // row range need the byte counts of a partial tile.
  const int pcc = tid & 15, pcol = tid >> 4;
  const double* pa = A + (j0 + pcol < n ? (j0 + pcol) * lda : 0) + kb + 2 * pcc;
  const int64_t pstride = 8 * lda;  // 8 columns
  uint32_t pvalid = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) pvalid |= (j0 + pcol + 8 * u < n) ? (1u << u) : 0u;
  const uint32_t pdst = pcol * kImColPitch + pcc * 16;
  const int8_t* po = O + (tid >> 1) * ld8 + kb + 16 * (tid & 1);
  const uint32_t podst = Cfg::kAStage + (tid >> 1) * kImOmPitch + (tid & 1) * 16;
  const bool all_cols = j0 + kImCols <= n;
  auto issue = [&](int s, uint32_t st) {
    const int64_t off = static_cast<int64_t>(s) * 32;
    if (all_cols && kb + off + 32 <= ke) {  // whole tile in range (all but the CTA's last k-step)
#pragma unroll
      for (int u = 0; u < 4; ++u) cp_async16(st + pdst + u * (8 * kImColPitch), pa + off + u * pstride, 16);
    } else {
      const int64_t rem = ke - (kb + off + 2 * pcc);  // rows left in this thread's chunk column
      const int full = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int bytes = ((pvalid >> u) & 1u) ? full : 0;
        cp_async16(st + pdst + u * (8 * kImColPitch), bytes ? pa + off + u * pstride : A, bytes);
      }
    }
    if (tid < 32 * MT) cp_async16(st + podst, po + off, 16);
  };

  for (int e = tid; e < kImWarps * 16 * MT * 8; e += kImThreads) yacc[e] = 0.0;
  __syncthreads();
  int acc[NS][MT][4];
#pragma unroll
  for (int t = 0; t < NS; ++t)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[t][mt][v] = 0;
  int ecol = 0;  // running exponent of this thread's B column (g); 0 = nothing seen yet
  uint32_t hlim = 1u << 20;  // values with exponent field > ecol have |hi word| >= hlim
  double asq4[4] = {0.0, 0.0, 0.0, 0.0};
  // 2^(1076 - E): fone when representable, else fa * fb (E = 1 until the first nonzero exponent:
  // columns of subnormals still convert exactly)
  double fa = pow2i((kSh - 1) / 2), fb = pow2i(kSh - 1 - (kSh - 1) / 2), fone = 1.0;
  bool two_step = true;
  double* yw = yacc + warp * (16 * MT * 8);  // [col 0..7][row 0..16*MT)

  // fold the int32 slices into the fp64 accumulators: C columns 2q, 2q+1 use their column's E
  auto flush = [&](int e_old) {
    const int e0 = max(__shfl_sync(0xffffffffu, e_old, (2 * q) * 4), 1);
    const int e1 = max(__shfl_sync(0xffffffffu, e_old, (2 * q + 1) * 4), 1);
    const int sh0 = e0 - kSh, sh1 = e1 - kSh;  // <= 970
    const double f0a = pow2i(sh0 / 2), f0b = pow2i(sh0 - sh0 / 2), f1a = pow2i(sh1 / 2), f1b = pow2i(sh1 - sh1 / 2);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        double s = static_cast<double>(acc[NS - 1][mt][v]);
#pragma unroll
        for (int t = NS - 2; t >= 0; --t) s = fma(s, 256.0, static_cast<double>(acc[t][mt][v]));
        const bool c1 = v & 1;
        s = s * (c1 ? f1a : f0a) * (c1 ? f1b : f0b);
        const int row = mt * 16 + g + 8 * (v >> 1), col = 2 * q + (v & 1);
        yw[col * (16 * MT) + row] += s;
#pragma unroll
        for (int t = 0; t < NS; ++t) acc[t][mt][v] = 0;
      }
  };

  uint32_t st_issue = 0, st_cur = 0;  // ring slots (byte offsets) of the next issue / the current k-step
#pragma unroll
  for (int s = 0; s < Cfg::kStages - 1; ++s) {
    if (s < nsteps) issue(s, sbase + st_issue);
    cp_async_commit();
    st_issue += Cfg::kStage;
  }
  // Software pipeline: the slices of k-step s+1 are formed while the MMAs of k-step s run (the
  // two instruction streams are independent unless a column's exponent grows, in which case the
  // MMAs of s complete, the accumulators are folded, then s+1 is converted with the new scale).
  auto load_x = [&](uint32_t slot, double (&x)[8]) {
    const double* colp = reinterpret_cast<const double*>(ims + slot + (8 * warp + g) * kImColPitch);
    const double2 p0 = *reinterpret_cast<const double2*>(colp + 4 * q);
    const double2 p1 = *reinterpret_cast<const double2*>(colp + 4 * q + 2);
    const double2 p2 = *reinterpret_cast<const double2*>(colp + 16 + 4 * q);
    const double2 p3 = *reinterpret_cast<const double2*>(colp + 16 + 4 * q + 2);
    x[0] = p0.x; x[1] = p0.y; x[2] = p1.x; x[3] = p1.y; x[4] = p2.x; x[5] = p2.y; x[6] = p3.x; x[7] = p3.y;
    // ||A||^2 and this thread's largest |hi word| (monotone in |x|); the column-wide exponent is
    // only formed (shuffles) on the rare path where some value reaches the current scale's limit
    uint32_t hmax = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      asq4[u & 3] = fma(x[u], x[u], asq4[u & 3]);
      hmax = max(hmax, static_cast<uint32_t>(__double2hiint(x[u])) & 0x7fffffffu);
    }
    return hmax;
  };
  auto column_emax = [&](uint32_t hmax) {
    int emax = static_cast<int>(hmax >> 20);
    emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, 1));
    return max(emax, __shfl_xor_sync(0xffffffffu, emax, 2));
  };
  auto rescale = [&](int emax) {
    ecol = max(ecol, emax + 1 < 2046 ? emax + 1 : emax);  // one bit of headroom: fewer flushes
    hlim = static_cast<uint32_t>(ecol + 1) << 20;          // |hi word| >= hlim <=> exponent > ecol
    const int sh = kSh - max(ecol, 1);
    fa = pow2i(sh / 2);
    fb = pow2i(sh - sh / 2);
    fone = pow2i(sh < 1023 ? sh : 0);
    two_step = __any_sync(0xffffffffu, sh >= 1023);
  };
  // w = rint(x * 2^(kSh - E)) (columns below 2^-969 scale in two exact steps); slices = its bytes
  auto convert = [&](const double (&x)[8], uint32_t (&b0)[kImSlices], uint32_t (&b1)[kImSlices]) {
    uint32_t lo[8], hi[8];
    if (!two_step) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long w = __double2ll_rn(x[u] * fone);
        lo[u] = static_cast<uint32_t>(w);
        hi[u] = static_cast<uint32_t>(static_cast<unsigned long long>(w) >> 32);
      }
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long w = __double2ll_rn((x[u] * fa) * fb);
        lo[u] = static_cast<uint32_t>(w);
        hi[u] = static_cast<uint32_t>(static_cast<unsigned long long>(w) >> 32);
      }
    }
    byte_transpose(lo[0], lo[1], lo[2], lo[3], hi[0], hi[1], hi[2], hi[3], b0);
    byte_transpose(lo[4], lo[5], lo[6], lo[7], hi[4], hi[5], hi[6], hi[7], b1);
  };
  // operator fragments (ldmatrix.x4 of 16 rows x 32 bytes per m-tile) x slices
  auto mma_step = [&](uint32_t slot, const uint32_t (&b0)[kImSlices], const uint32_t (&b1)[kImSlices]) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      uint32_t af[4];
      const int r = mt * 16 + (lane & 15);
      const uint32_t addr = sbase + slot + Cfg::kAStage + r * kImOmPitch + (lane >> 4) * 16;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                   : "=r"(af[0]), "=r"(af[1]), "=r"(af[2]), "=r"(af[3])
                   : "r"(addr));
#pragma unroll
      for (int t = 0; t < NS - 1; ++t) imma_16x8x32<false>(acc[t][mt], af, b0[t], b1[t]);
      imma_16x8x32<true>(acc[NS - 1][mt], af, b0[NS - 1], b1[NS - 1]);
    }
  };
  auto next_slot = [&](uint32_t v) { return v + Cfg::kStage == Cfg::kStages * Cfg::kStage ? 0u : v + Cfg::kStage; };

  uint32_t bc0[kImSlices], bc1[kImSlices];  // slices of the current k-step
  if (nsteps > 0) {
    cp_async_wait<Cfg::kStages - 2>();
    __syncthreads();
    double x[8];
    const uint32_t hmax = load_x(st_cur, x);
    if (__any_sync(0xffffffffu, hmax >= hlim)) rescale(column_emax(hmax));  // nothing accumulated yet
    convert(x, bc0, bc1);
  }
  for (int s = 0; s < nsteps; ++s) {
    cp_async_wait<Cfg::kStages - 3>();  // k-step s + 1 has landed
    __syncthreads();                 // and every warp is done with k-step s - 1's slot
    if (s + Cfg::kStages - 1 < nsteps) issue(s + Cfg::kStages - 1, sbase + st_issue);
    cp_async_commit();
    st_issue = next_slot(st_issue);
    const uint32_t cur = st_cur;
    st_cur = next_slot(st_cur);
    if (s + 1 < nsteps) {
      double x[8];
      const uint32_t hmax = load_x(st_cur, x);
      uint32_t bn0[kImSlices], bn1[kImSlices];
      if (!__any_sync(0xffffffffu, hmax >= hlim)) {
        convert(x, bn0, bn1);  // independent of the MMAs below: the scheduler interleaves them
        mma_step(cur, bc0, bc1);
      } else {
        mma_step(cur, bc0, bc1);
        const int emax = column_emax(hmax);
        flush(ecol);
        rescale(emax);
        convert(x, bn0, bn1);
      }
#pragma unroll
      for (int t = 0; t < kImSlices; ++t) {
        bc0[t] = bn0[t];
        bc1[t] = bn1[t];
      }
    } else {
      mma_step(cur, bc0, bc1);
    }
  }
  cp_async_wait<0>();
  flush(ecol);
  __syncwarp();
  // write this split's partial: Y(h, j) at part[split][j * c_pad + h]
  double* out = part + static_cast<int64_t>(blockIdx.y) * split_stride;
  for (int e = lane; e < 8 * 16 * MT; e += 32) {
    const int col = e / (16 * MT), row = e - col * (16 * MT);
    const int64_t j = j0 + 8 * warp + col;
    if (j < n && row < c_pad) out[j * c_pad + row] = yw[e];
  }
  const double bs = block_sum<kImThreads>((asq4[0] + asq4[1]) + (asq4[2] + asq4[3]), red);
  if (tid == 0) asq_part[blockIdx.y * gridDim.x + blockIdx.x] = bs;
}

bool sparse_sketch_imma_supported(const double* A, int64_t lda, int64_t c_pad) {
  return c_pad <= 64 && (lda % 2) == 0 && (reinterpret_cast<uintptr_t>(A) % 16) == 0;
}

struct ImPlan {
  int64_t col_tiles, splits, kps, ld8, mt;
};
static ImPlan plan_imma(int64_t m, int64_t n, int64_t c_pad) {
  ImPlan p{};
  p.mt = (c_pad + 15) / 16;
  p.col_tiles = ceil_div(n, kImCols);
  const int64_t steps = ceil_div(m, 32);
  // enough CTAs for 2 per SM x a few waves; at least 64 k-steps per split; <= 2^17 k-steps per
  // split keeps every int32 slice sum exact (|acc| <= 32 * 255 per k-step)
  const int64_t want = 148 * 2 * 4;
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>(ceil_div(want, p.col_tiles), steps / 64));
  splits = std::max<int64_t>(splits, ceil_div(steps, int64_t(1) << 17));
  p.kps = ceil_div(steps, splits);
  p.splits = ceil_div(steps, p.kps);
  p.ld8 = round_up(std::max<int64_t>(m, 1) + 32, 32);  // one k-step of zero padding past m
  return p;
}

int64_t sparse_sketch_imma_workspace_elems(int64_t m, int64_t n, int64_t c_pad) {
  const ImPlan p = plan_imma(m, n, c_pad);
  const int64_t part = p.splits > 1 ? p.splits * n * c_pad : 0;
  const int64_t om = ceil_div(16 * p.mt * p.ld8, 8);
  return part + p.col_tiles * p.splits + om + 4096 + 8;
}

cudaError_t run_sketch_apply_sparse_imma(const double* A, int64_t m, int64_t n, int64_t lda, uint64_t seed, int64_t c,
                                         int64_t c_pad, int zeta, double scale, double* Y, double* ws, int64_t ws_elems,
                                         const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info,
                                         bool operator_ready, bool kernel_only) {
  if (!sparse_sketch_imma_supported(A, lda, c_pad)) return cudaErrorInvalidValue;
  const ImPlan p = plan_imma(m, n, c_pad);
  if (sparse_sketch_imma_workspace_elems(m, n, c_pad) > ws_elems) return cudaErrorInvalidValue;
  const int64_t part_elems = p.splits > 1 ? p.splits * n * c_pad : 0;
  double* part = ws;
  double* asq_part = ws + part_elems;
  int8_t* O = reinterpret_cast<int8_t*>(round_up(reinterpret_cast<uintptr_t>(asq_part + p.col_tiles * p.splits), 64));
  double* ysq_part = reinterpret_cast<double*>(O + 16 * p.mt * p.ld8);
  ysq_part = reinterpret_cast<double*>(round_up(reinterpret_cast<uintptr_t>(ysq_part), 16));
  cudaError_t e;
  if (!operator_ready) {
    e = cudaMemsetAsync(O, 0, static_cast<size_t>(16 * p.mt * p.ld8), st);
    if (e != cudaSuccess) return e;
    const int ze = static_cast<int>(std::min<int64_t>(zeta, c));
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(m, 256), 148 * 16));
    gen_sparse_sign_i8_kernel<<<blocks, 256, 0, st>>>(O, p.ld8, c, m, seed, ze);
  }
  auto launch = [&](auto kern, int smem) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    dim3 grid(static_cast<unsigned>(p.col_tiles), static_cast<unsigned>(p.splits));
    kern<<<grid, kImThreads, smem, st>>>(A, m, n, lda, O, p.ld8, p.kps, c_pad, p.splits > 1 ? part : Y, n * c_pad,
                                         asq_part);
    return cudaGetLastError();
  };
  const int ns_env = getenv("ITERCUR_IMMA_SLICES") ? atoi(getenv("ITERCUR_IMMA_SLICES")) : 0;  // A/B
  const int ns = ns_env == 6 || ns_env == 7 ? ns_env : (p.mt <= 2 ? 7 : 6);
  switch (p.mt * 10 + ns) {
    case 17: e = launch(sparse_sketch_imma_kernel<1, 7>, ImCfg<1>::kSmem); break;
    case 16: e = launch(sparse_sketch_imma_kernel<1, 6>, ImCfg<1>::kSmem); break;
    case 27: e = launch(sparse_sketch_imma_kernel<2, 7>, ImCfg<2>::kSmem); break;
    case 26: e = launch(sparse_sketch_imma_kernel<2, 6>, ImCfg<2>::kSmem); break;
    case 37: e = launch(sparse_sketch_imma_kernel<3, 7>, ImCfg<3>::kSmem); break;
    case 36: e = launch(sparse_sketch_imma_kernel<3, 6>, ImCfg<3>::kSmem); break;
    case 47: e = launch(sparse_sketch_imma_kernel<4, 7>, ImCfg<4>::kSmem); break;
    default: e = launch(sparse_sketch_imma_kernel<4, 6>, ImCfg<4>::kSmem); break;
  }
  if (e != cudaSuccess) return e;
  if (info) {
    info->splits = static_cast<int>(p.splits);
    info->ctas = static_cast<int>(p.col_tiles * p.splits);
    info->nt = static_cast<int>(p.mt);
    info->tma = false;
    info->dominant_launches = 1;
  }
  if (kernel_only) return cudaGetLastError();
  const int64_t total = n * c_pad;
  const int rblocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 2048));
  sketch_reduce_kernel<<<rblocks, 256, 0, st>>>(p.splits > 1 ? part : Y, p.splits > 1 ? static_cast<int>(p.splits) : 1,
                                                n * c_pad, scale, Y, total, ysq_part);
  reduce_partials_kernel<<<1, 256, 0, st>>>(ysq_part, rblocks, stats.d_ysq);
  reduce_partials_kernel<<<1, 256, 0, st>>>(asq_part, static_cast<int>(p.col_tiles * p.splits), stats.d_asq);
  return cudaGetLastError();
}


// ------------------------------------------------------------------ sparse-sign sketch, tcgen05 form
// The same sliced-integer contraction as sparse_sketch_imma_kernel, on the 5th-generation tensor
// cores: tcgen05.mma kind::i8 with the int32 slice accumulators in TMEM instead of registers.
//   D (128 columns of A x NPAD sketch rows, s32, TMEM) += slices_t (128 x 32 rows, u8/s8, smem)
//                                                        x Omega^T (32 rows x NPAD, s8, smem)
// for t = 0..NS-1 into TMEM columns [t*NPAD, (t+1)*NPAD). Warp roles (192 threads):
//   warps 0-3  conversion: thread = one column of the CTA's 128; reads its 32 doubles of the
//              k-step from the TMA tile (two 16-row boxes, 128-B swizzle), forms
//              w = rint(x * 2^(kSh - E)) against its column's running exponent E, writes the NS
//              byte slices in the canonical K-major no-swizzle layout (8-row x 16-byte core
//              matrices), and when its column's exponent grows folds its TMEM lane into FP64
//              registers (tcgen05.ld), zeroes it (tcgen05.st) and rescales — per warp, no
//              CTA-wide coupling;
//   warp 4     producer: TMA of the A tile (2 boxes) + bulk copy of the k-step's operator block;
//   warp 5     one thread issues the NS MMAs per k-step and commits them to mbarriers.
// Rings: A/operator stages (full: TMA bytes; empty: 128 conversion arrivals + 1 MMA commit) and
// double-buffered slice tiles (full: 128 arrivals; empty: MMA commit).
constexpr int kUmThreads = 320;  // 8 converter warps + producer + MMA issuer
constexpr int kUmCols = 128;               // MMA M: columns of A per CTA (one TMEM lane each)
constexpr int kUmABytes = kUmCols * 32 * 8;  // 32 KB per k-step (two 16-row TMA boxes)

template <int NPAD>
struct UmCfg {
  static constexpr int kNS = NPAD == 32 ? 7 : 6;      // slices (TMEM: NS*NPAD accumulators + 2*NS*8 operand)
  static constexpr int kOBytes = NPAD * 32;           // operator block per k-step
  static constexpr int kTmemCols = 512;
  static constexpr int kStages = 4;                   // A / operator ring
  static constexpr int kYaccBytes = NPAD * kUmCols * 8;
  static constexpr int kSmem = kStages * (kUmABytes + kOBytes) + kYaccBytes + 2048 + 256 + 1024;
  static_assert(kNS * NPAD + 2 * kNS * 8 <= kTmemCols, "TMEM budget");
};

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  // K-major, no swizzle: core matrices of 8 rows x 16 B (128 B contiguous); the two K halves 128 B
  // apart (LBO), consecutive 8-row groups 256 B apart (SBO); version 1 (sm_100)
  return static_cast<uint64_t>((saddr >> 4) & 0x3fffu) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(256 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint32_t umma_idesc_i8(bool a_signed, int n) {
  // c = s32 (2), a = u8/s8, b = s8 (operator), both K-major, N >> 3, M = 128 >> 4
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(128 >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc ? 1 : 0));
}
// A operand from TMEM (128 lanes x 8 columns: row = lane, bytes k = 4c..4c+3 in column c)
__device__ __forceinline__ void umma_i8_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc ? 1 : 0));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16_zero(uint32_t taddr) {
  const uint32_t z = 0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr),
      "r"(z)
      : "memory");
}

template <int NPAD, int NS>
__global__ void __launch_bounds__(kUmThreads, 1)
    sparse_sketch_umma_kernel(const __grid_constant__ CUtensorMap tmA, const int8_t* __restrict__ Oblk, int64_t m,
                              int64_t n, int64_t col_tiles, int64_t items, int64_t kps, int64_t c_pad,
                              double* __restrict__ part, int64_t split_stride, double* __restrict__ asq_part,
                              int ablate) {
  // Persistent: CTA b processes work items b, b + gridDim.x, ... (item = split * col_tiles + column
  // tile); the rings and their phases run on across items, so the producer prefetches the next
  // item's tiles while the converters fold the finished one.
  using Cfg = UmCfg<NPAD>;
  constexpr int kSh = 1076 - 8 * (7 - NS);
  extern __shared__ __align__(1024) uint8_t ums[];
  uint8_t* sA = ums;                                             // Cfg::kStages x 32 KB (1024-aligned)
  uint8_t* sO = sA + Cfg::kStages * kUmABytes;                      // Cfg::kStages x operator block
  double* yacc = reinterpret_cast<double*>(sO + Cfg::kStages * Cfg::kOBytes);  // [NPAD][128] FP64 sums
  uint32_t* hx = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(yacc) + Cfg::kYaccBytes);  // [2][2][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(hx + 512);
  uint64_t* empty = full + Cfg::kStages;
  uint64_t* sfull = empty + Cfg::kStages;
  uint64_t* sempty = sfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 2);
  __shared__ double red[8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto item_range = [&](int64_t it, int64_t& j0, int64_t& kb, int& nsteps) {
    const int64_t ct = it % col_tiles, sp = it / col_tiles;
    j0 = ct * kUmCols;
    kb = sp * kps * 32;
    const int64_t ke = m < kb + kps * 32 ? m : kb + kps * 32;
    nsteps = static_cast<int>(ke > kb ? (ke - kb + 31) / 32 : 0);
  };

  if (tid == 0) {
    for (int q = 0; q < Cfg::kStages; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], 2 * kUmCols + 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(&sfull[q], 2 * kUmCols);
      mbar_init(&sempty[q], 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(Cfg::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ---------------- producer
    if (lane == 0) {
      prefetch_tmap(&tmA);
      int64_t g = 0;
      for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        int64_t j0, kb;
        int nsteps;
        item_range(it, j0, kb, nsteps);
        for (int s = 0; s < nsteps; ++s, ++g) {
          const int st = static_cast<int>(g % Cfg::kStages);
          if (g >= Cfg::kStages) mbar_wait(&empty[st], static_cast<uint32_t>((g / Cfg::kStages) - 1) & 1);
          mbar_arrive_expect_tx(&full[st], kUmABytes + Cfg::kOBytes);
          const int32_t r0 = static_cast<int32_t>(kb + 32 * s);
          tma_load_2d(sA + st * kUmABytes, &tmA, &full[st], r0, static_cast<int32_t>(j0));
          tma_load_2d(sA + st * kUmABytes + kUmABytes / 2, &tmA, &full[st], r0 + 16, static_cast<int32_t>(j0));
          bulk_g2s(sO + st * Cfg::kOBytes, Oblk + (kb / 32 + s) * Cfg::kOBytes, Cfg::kOBytes, &full[st]);
        }
      }
    }
  } else if (warp == 9) {
    // ---------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc_u = umma_idesc_i8(false, NPAD), idesc_s = umma_idesc_i8(true, NPAD);
      int64_t g = 0;
      for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        int64_t j0, kb;
        int nsteps;
        item_range(it, j0, kb, nsteps);
        for (int s = 0; s < nsteps; ++s, ++g) {
          const int st = static_cast<int>(g % Cfg::kStages), sb = static_cast<int>(g & 1);
          mbar_wait(&full[st], static_cast<uint32_t>(g / Cfg::kStages) & 1);
          mbar_wait(&sfull[sb], static_cast<uint32_t>(g >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint64_t bdesc = umma_desc(smem_u32(sO + st * Cfg::kOBytes));
          if (!(ablate & 2)) {
#pragma unroll
            for (int t = 0; t < NS; ++t)
              umma_i8_ta(tmem + t * NPAD, tmem + NS * NPAD + (sb * NS + t) * 8, bdesc, t == NS - 1 ? idesc_s : idesc_u,
                         s > 0);
          }
          umma_commit(&sempty[sb]);  // the slice tile may be rewritten once these MMAs are done
          umma_commit(&empty[st]);   // the operator block is consumed (the A tile by the converters)
        }
      }
    }
  } else {
    // ---------------- conversion (warps 0-7): thread = rows 16*half.. of column jl of the item's 128;
    // warps w and w + 4 share columns (and TMEM lanes 32*(w%4)..); the column exponent is their
    // joint maximum (exchanged through shared memory), the TMEM fold is done by the half-0 warp
    const int cw = warp & 3, half = warp >> 2;
    const int jl = cw * 32 + lane;
    const uint32_t tl = tmem + (static_cast<uint32_t>(32 * cw) << 16);  // this warp's TMEM lanes
    const uint32_t my_off = static_cast<uint32_t>(jl) * 128u;
    int64_t g = 0;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      int64_t j0, kb;
      int nsteps;
      item_range(it, j0, kb, nsteps);
#pragma unroll 8
      for (int h = 0; h < NPAD; ++h) yacc[h * kUmCols + jl] = 0.0;
      double asq4[4] = {0.0, 0.0, 0.0, 0.0};
      int ecol = 0;
      uint32_t hlim = 1u << 20;
      double fa = pow2i((kSh - 1) / 2), fb = pow2i(kSh - 1 - (kSh - 1) / 2), fone = 1.0;
      bool two_step = true;
      // fold this warp's TMEM lanes (all slices) into yacc with the current scale, then zero them
      auto fold = [&]() {
        const int sh = max(ecol, 1) - kSh;  // <= 970
#pragma unroll
        for (int t = 0; t < NS; ++t) {
          const int e = sh + 8 * t;
          const double f1 = pow2i(e / 2), f2 = pow2i(e - e / 2);
#pragma unroll
          for (int c0 = 0; c0 < NPAD; c0 += 16) {
            uint32_t r[16];
            tmem_ld16(tl + t * NPAD + c0, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int v = 0; v < 16; ++v)
              yacc[(c0 + v) * kUmCols + jl] += (static_cast<double>(static_cast<int>(r[v])) * f1) * f2;
            tmem_st16_zero(tl + t * NPAD + c0);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      };
      for (int s = 0; s < nsteps; ++s, ++g) {
        const int st = static_cast<int>(g % Cfg::kStages), sb = static_cast<int>(g & 1);
        mbar_wait(&full[st], static_cast<uint32_t>(g / Cfg::kStages) & 1);
        double x[16];
        const uint8_t* tile = sA + st * kUmABytes + half * (kUmABytes / 2);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double2 v = *reinterpret_cast<const double2*>(tile + my_off + (((c ^ (jl & 7)) & 7) << 4));
          x[2 * c] = v.x;
          x[2 * c + 1] = v.y;
        }
        mbar_arrive(&empty[st]);  // A tile consumed (values are in registers)
        if (ablate & 1) {  // measurement only: stream the tiles, skip the conversion
          asq4[0] += x[0] + x[15];
          if (g >= 2) mbar_wait(&sempty[sb], static_cast<uint32_t>((g >> 1) - 1) & 1);
          mbar_arrive(&sfull[sb]);
          continue;
        }
        uint32_t hmax = 0;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          asq4[u & 3] = fma(x[u], x[u], asq4[u & 3]);
          hmax = max(hmax, static_cast<uint32_t>(__double2hiint(x[u])) & 0x7fffffffu);
        }
        uint32_t* hxs = hx + (g & 1) * 256;
        hxs[half * 128 + jl] = hmax;
        asm volatile("bar.sync %0, 64;\n" ::"r"(2 + cw) : "memory");
        hmax = max(hmax, hxs[(half ^ 1) * 128 + jl]);
        // the slice buffer sb (TMEM) is free once the MMAs of global k-step g - 2 are done
        if (g >= 2) mbar_wait(&sempty[sb], static_cast<uint32_t>((g >> 1) - 1) & 1);
        if (__any_sync(0xffffffffu, hmax >= hlim)) {
          if (s >= 1 && half == 0) {  // the MMAs of k-step g - 1 complete before this warp reads its lanes
            mbar_wait(&sempty[sb ^ 1], static_cast<uint32_t>((g - 1) >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            fold();
          }
          const int emax = static_cast<int>(hmax >> 20);
          if (emax > ecol) {
            ecol = emax + 1 < 2046 ? emax + 1 : emax;
            hlim = static_cast<uint32_t>(ecol + 1) << 20;
          }
          const int sh = kSh - max(ecol, 1);
          fa = pow2i(sh / 2);
          fb = pow2i(sh - sh / 2);
          fone = pow2i(sh < 1023 ? sh : 0);
          two_step = sh >= 1023;
        }
        // scale (one multiply; columns below 2^-969 take two exact steps on a warp-uniform slow path)
        if (__any_sync(0xffffffffu, two_step)) {
#pragma unroll
          for (int u = 0; u < 16; ++u) x[u] = two_step ? (x[u] * fa) * fb : x[u] * fone;
        } else {
#pragma unroll
          for (int u = 0; u < 16; ++u) x[u] *= fone;
        }
        // slices -> the MMA's A operand in TMEM: lane = column, this half's 16 bytes of slice t in
        // columns NS*NPAD + (sb*NS + t)*8 + 4*half .. +3 (4 rows per 32-bit column)
        uint32_t sl[2][NS][2];
#pragma unroll
        for (int g8 = 0; g8 < 2; ++g8) {
          uint32_t lo[8], hi[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const long long w = __double2ll_rn(x[8 * g8 + u]);
            lo[u] = static_cast<uint32_t>(w);
            hi[u] = static_cast<uint32_t>(static_cast<unsigned long long>(w) >> 32);
          }
          uint32_t b0[kImSlices], b1[kImSlices];
          byte_transpose(lo[0], lo[1], lo[2], lo[3], hi[0], hi[1], hi[2], hi[3], b0);
          byte_transpose(lo[4], lo[5], lo[6], lo[7], hi[4], hi[5], hi[6], hi[7], b1);
#pragma unroll
          for (int t = 0; t < NS; ++t) {
            sl[g8][t][0] = b0[t];
            sl[g8][t][1] = b1[t];
          }
        }
        const uint32_t ta = tl + NS * NPAD + sb * NS * 8 + 4 * half;
#pragma unroll
        for (int t = 0; t < NS; ++t) tmem_st4(ta + 8 * t, sl[0][t][0], sl[0][t][1], sl[1][t][0], sl[1][t][1]);
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        mbar_arrive(&sfull[sb]);
      }
      // item done: fold after its last MMAs, write the split's partial column, ||A||^2 partial
      if (nsteps > 0 && half == 0) {
        mbar_wait(&sempty[(g - 1) & 1], static_cast<uint32_t>((g - 1) >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        fold();
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      }
      const int64_t j = j0 + jl;
      if (half == 0 && j < n) {
        double* out = part + (it / col_tiles) * split_stride + j * c_pad;
#pragma unroll 8
        for (int h = 0; h < NPAD; ++h)
          if (h < c_pad) out[h] = yacc[h * kUmCols + jl];
      }
      const double ws = warp_sum((asq4[0] + asq4[1]) + (asq4[2] + asq4[3]));
      if (lane == 0) red[warp] = ws;
      asm volatile("bar.sync 1, 256;\n" ::: "memory");
      if (tid == 0) asq_part[it] = ((red[0] + red[1]) + (red[2] + red[3])) + ((red[4] + red[5]) + (red[6] + red[7]));
      asm volatile("bar.sync 1, 256;\n" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(Cfg::kTmemCols) : "memory");
  }
}

// operator in per-k-step blocks of the canonical K-major layout: block q (rows 32q..32q+31 of A)
// holds Omega(h, 32q + kk) at ((h / 8) * 2 + kk / 16) * 128 + (h % 8) * 16 + kk % 16
__global__ void gen_sparse_sign_umma_kernel(int8_t* O, int npad, int64_t c, int64_t m, uint64_t seed, int zeta_eff) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t rows[16];
    int8_t signs[16];
    sparse_sign_slots(seed, i, c, zeta_eff, rows, signs);
    const int64_t q = i >> 5;
    const int kk = static_cast<int>(i & 31);
    int8_t* blk = O + q * npad * 32;
    for (int t = 0; t < zeta_eff; ++t) {
      const int h = rows[t];
      blk[((h >> 3) * 2 + (kk >> 4)) * 128 + (h & 7) * 16 + (kk & 15)] = signs[t];
    }
  }
}

bool sparse_sketch_umma_supported(const double* A, int64_t m, int64_t n, int64_t lda, int64_t c_pad) {
  return c_pad <= 64 && (lda % 2) == 0 && (reinterpret_cast<uintptr_t>(A) % 16) == 0 && m < (int64_t(1) << 31) &&
         n < (int64_t(1) << 31);
}

struct UmPlan {
  int64_t col_tiles, splits, kps, npad, ksteps, items, grid;
};
static int num_sms() {
  static int sms = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return sms;
}
static UmPlan plan_umma(int64_t m, int64_t n, int64_t c_pad) {
  UmPlan p{};
  p.npad = c_pad <= 32 ? 32 : 64;
  p.col_tiles = ceil_div(n, kUmCols);
  p.ksteps = ceil_div(m, 32);
  const int64_t sms = num_sms();
  // persistent CTAs (one per SM): the split count minimising the busiest CTA's k-steps, charging each
  // item ~8 k-steps of fold/drain and each split a partial Y pass; >= 32 k-steps per item; <= 2^17
  // k-steps per item keeps every int32 slice sum exact
  int64_t s = 1;
  double best = 1e300;
  for (int64_t t = 1; t <= 64; ++t) {
    const int64_t kps = ceil_div(p.ksteps, t);
    if (t > 1 && kps < 32) break;
    const int64_t items = p.col_tiles * ceil_div(p.ksteps, kps);
    const double per_cta = std::ceil(static_cast<double>(items) / sms) * (kps + 8.0);
    const double partials = t > 1 ? 2.0 * t * n * c_pad * 8.0 / (32.0 * kUmCols * 8.0 * sms) : 0.0;
    if (per_cta + partials < best) {
      best = per_cta + partials;
      s = t;
    }
  }
  if (const char* e = getenv("ITERCUR_UMMA_SPLITS")) s = std::max<int64_t>(1, atoll(e));  // A/B
  s = std::max<int64_t>(s, ceil_div(p.ksteps, int64_t(1) << 17));
  p.kps = ceil_div(p.ksteps, s);
  p.splits = ceil_div(p.ksteps, p.kps);
  p.items = p.col_tiles * p.splits;
  p.grid = std::min<int64_t>(p.items, sms);
  return p;
}

int64_t sparse_sketch_umma_workspace_elems(int64_t m, int64_t n, int64_t c_pad) {
  const UmPlan p = plan_umma(m, n, c_pad);
  const int64_t part = p.splits > 1 ? p.splits * n * c_pad : 0;
  const int64_t om = ceil_div(p.ksteps * p.npad * 32, 8);
  return part + p.items + om + 4096 + 16;
}

cudaError_t run_sketch_apply_sparse_umma(const double* A, int64_t m, int64_t n, int64_t lda, uint64_t seed, int64_t c,
                                         int64_t c_pad, int zeta, double scale, double* Y, double* ws, int64_t ws_elems,
                                         const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info,
                                         bool operator_ready, bool kernel_only) {
  if (!sparse_sketch_umma_supported(A, m, n, lda, c_pad)) return cudaErrorInvalidValue;
  const UmPlan p = plan_umma(m, n, c_pad);
  if (sparse_sketch_umma_workspace_elems(m, n, c_pad) > ws_elems) return cudaErrorInvalidValue;
  const int64_t part_elems = p.splits > 1 ? p.splits * n * c_pad : 0;
  double* part = ws;
  double* asq_part = ws + part_elems;
  int8_t* O = reinterpret_cast<int8_t*>(round_up(reinterpret_cast<uintptr_t>(asq_part + p.items), 128));
  double* ysq_part = reinterpret_cast<double*>(round_up(reinterpret_cast<uintptr_t>(O + p.ksteps * p.npad * 32), 16));
  cudaError_t e;
  if (!operator_ready) {
    e = cudaMemsetAsync(O, 0, static_cast<size_t>(p.ksteps * p.npad * 32), st);
    if (e != cudaSuccess) return e;
    const int ze = static_cast<int>(std::min<int64_t>(zeta, c));
    const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(m, 256), 148 * 16));
    gen_sparse_sign_umma_kernel<<<blocks, 256, 0, st>>>(O, static_cast<int>(p.npad), c, m, seed, ze);
  }
  CUtensorMap tmA{};
  if (!make_tmap_2d(&tmA, A, m, n, lda, 16, kUmCols)) return cudaErrorInvalidValue;
  auto launch = [&](auto kern, int npad) {
    const int smem = npad == 32 ? UmCfg<32>::kSmem : UmCfg<64>::kSmem;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    const int ablate = getenv("ITERCUR_UMMA_ABLATE") ? atoi(getenv("ITERCUR_UMMA_ABLATE")) : 0;  // measurement
    kern<<<static_cast<unsigned>(p.grid), kUmThreads, smem, st>>>(tmA, O, m, n, p.col_tiles, p.items, p.kps, c_pad,
                                                                   p.splits > 1 ? part : Y, n * c_pad, asq_part,
                                                                   ablate);
    return cudaGetLastError();
  };
  if (p.npad == 32) e = launch(sparse_sketch_umma_kernel<32, UmCfg<32>::kNS>, 32);
  else e = launch(sparse_sketch_umma_kernel<64, UmCfg<64>::kNS>, 64);
  if (e != cudaSuccess) return e;
  if (info) {
    info->splits = static_cast<int>(p.splits);
    info->ctas = static_cast<int>(p.grid);
    info->nt = static_cast<int>(p.npad);
    info->tma = true;
    info->dominant_launches = 1;
  }
  if (kernel_only) return cudaGetLastError();
  const int64_t total = n * c_pad;
  const int rblocks = static_cast<int>(std::min<int64_t>(ceil_div(total, 256), 2048));
  sketch_reduce_kernel<<<rblocks, 256, 0, st>>>(p.splits > 1 ? part : Y, p.splits > 1 ? static_cast<int>(p.splits) : 1,
                                                n * c_pad, scale, Y, total, ysq_part);
  reduce_partials_kernel<<<1, 256, 0, st>>>(ysq_part, rblocks, stats.d_ysq);
  reduce_partials_kernel<<<1, 256, 0, st>>>(asq_part, static_cast<int>(p.items), stats.d_asq);
  return cudaGetLastError();
}

// a kernel of this translation unit (module), for itercur_preload
const void* module_anchor_sketch() { return reinterpret_cast<const void*>(gen_gaussian_kernel); }

}  // namespace itercur_b200

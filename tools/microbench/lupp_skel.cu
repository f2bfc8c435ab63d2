// Per-step cost of the cluster LUPP exchange skeleton (16 CTAs x 512 threads), with phases
// switched on/off by MODE bits, to find where the per-step latency goes.
//   bit0: compute warps do a warp argmax + tail write     bit1: service warps CTA argmax
//   bit2: push header+tail with st.async to every CTA      bit3: exchange warp argmax + copy
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct WCand { uint64_t key; int32_t idx; double second; };
__device__ __forceinline__ uint64_t mag_key(double m) { return static_cast<uint64_t>(__double_as_longlong(m)) + 1ull; }
__device__ __forceinline__ double key_mag(uint64_t k) { return k ? __longlong_as_double(static_cast<long long>(k - 1ull)) : -1.0; }
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}
__device__ __forceinline__ WCand warp_argmax(const WCand& c) {
  const uint64_t best = warp_max_u64(c.key);
  const int32_t tie = (c.key == best && best != 0) ? c.idx : 0x7fffffff;
  const int32_t widx = __reduce_min_sync(0xffffffffu, tie);
  const bool win = best != 0 && c.key == best && c.idx == widx;
  const double offer = win ? c.second : key_mag(c.key);
  const uint64_t sec = warp_max_u64(offer >= 0.0 ? mag_key(offer) : 0ull);
  return WCand{best, best ? widx : -1, key_mag(sec)};
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void st_async_v2(uint32_t ra, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(ra), "d"(a), "d"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
  return ok;
}

__device__ __noinline__ double ieee_div(double a, double p) { return __ddiv_rn(a, p); }
template <int MODE>
__global__ void __launch_bounds__(512, 1) skel(long long* out, int steps, double* rec) {
  constexpr int kWarps = 16, kSvc = 4, kComp = 12, SMAX = 20, SL = 26;
  __shared__ WCand wc[kComp];
  __shared__ WCand s_best[2];
  __shared__ __align__(16) double wtail[kComp][SMAX];
  __shared__ __align__(16) double inbox[2][16][SL];
  __shared__ double U[SMAX][SMAX];
  extern __shared__ double Ws[];  // [SMAX][800] (dynamic)
  double cur[2] = {1.0 + threadIdx.x * 1e-3, 2.0 + threadIdx.x * 1e-3};
  double fp[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ double s_rcp[2];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = cl.num_blocks(), me = cl.block_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&mbar[0], 1); mbar_init(&mbar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  if (threadIdx.x < 2 * 16 * SL) (&inbox[0][0][0])[threadIdx.x] = 0.0;
  for (int e = threadIdx.x; e < SMAX * 800; e += 512) Ws[e] = 1.0 + e * 1e-6;
  for (int e = threadIdx.x; e < SMAX * SMAX; e += 512) (&U[0][0])[e] = 0.5 + e * 1e-3;
  __syncthreads();
  cl.sync();
  const int npairs = 2 + SMAX / 2;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int col = s + 1, par = col & 1;
    const WCand bprev = s_best[s & 1];
    if ((MODE & 4) && warp == 0 && lane == 0) expect_tx(&mbar[par], static_cast<uint32_t>(CL * npairs * 16));
    if (warp >= kSvc) {
      const int cw = warp - kSvc;
      WCand mine{mag_key(1.0 + ((me * 977 + cw * 131 + lane * 17 + s * 7 + (int)(bprev.key & 3)) % 1009) * 1e-3),
                 me * 10000 + cw * 32 + lane, -1.0};
      if (MODE & 16) {
        // real row work: 2 rows per thread, Markstein quotient, 4-term panel update, merge
        const double pivot = U[s % SMAX][s % SMAX] + 1.5, y = 1.0 / pivot;
        double ucol[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) ucol[j] = U[j][(s + 1) % SMAX];
        mine = WCand{0ull, -1, -1.0};
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int rr = (cw * 32 + lane) + k * 384;
          const double x = cur[k];
          const double q0 = __dmul_rn(x, y);
          const double rm = __fma_rn(-q0, pivot, x);
          double f = __fma_rn(rm, y, q0);
          if (MODE & 128) {
            const double aq = fabs(f), ax = fabs(x);
            const bool bad = !(aq > 0x1p-968 && aq < 0x1p968 && ax > 0x1p-968 && ax < 0x1p968);
            if (__any_sync(0xffffffffu, bad)) f = ieee_div(x, pivot);
          }
          fp[k][s & 3] = f;
          double v = Ws[((s + 1) % SMAX) * 800 + rr];
#pragma unroll
          for (int j = 0; j < 4; ++j) if (j <= (s & 3)) v = __dsub_rn(v, __dmul_rn(fp[k][j], ucol[j]));
          Ws[(s % SMAX) * 800 + rr] = f;
          cur[k] = v;
          const uint64_t key = mag_key(fabs(v));
          const bool better = key > mine.key;
          mine.second = better ? key_mag(mine.key) : fmax(mine.second, fabs(v));
          mine.key = better ? key : mine.key;
          mine.idx = better ? me * 10000 + rr : mine.idx;
        }
      }
      WCand w = mine;
      if (MODE & 1) {
        w = warp_argmax(mine);
        if (MODE & 32) {
          const int lr = (w.idx < 0 ? 0 : w.idx % 10000), kw = lr / 384;
          double fw[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) fw[j] = __shfl_sync(0xffffffffu, kw ? fp[1][j] : fp[0][j], lr & 31);
          for (int t = s + 1 + lane; t < SMAX; t += 32) {
            double xx = Ws[t * 800 + lr % 800];
#pragma unroll
            for (int j = 0; j < 4; ++j) if (j <= (s & 3)) xx = __dsub_rn(xx, __dmul_rn(fw[j], U[j][t]));
            wtail[cw][t] = xx;
          }
        } else if (lane < SMAX) {
          wtail[cw][lane] = key_mag(w.key) + lane;
        }
      }
      if (lane == 0) wc[cw] = w;
    }
    __syncthreads();
    if (warp < kSvc) {
      WCand bc = lane < kComp ? wc[lane] : WCand{0ull, -1, -1.0};
      if (MODE & 2) bc = warp_argmax(bc);
      else bc = WCand{__shfl_sync(0xffffffffu, bc.key, 0), __shfl_sync(0xffffffffu, bc.idx, 0), -1.0};
      if ((MODE & 4) && lane < npairs) {
        double v0 = lane == 0 ? key_mag(bc.key) : (lane == 1 ? __longlong_as_double((long long)bc.idx) : 0.0);
        double v1 = lane == 0 ? bc.second : 0.0;
        if (lane >= 2) { const int ow = ((bc.idx < 0 ? 0 : bc.idx) % 10000) / 32 % kComp; v0 = wtail[ow][2 * (lane - 2)]; v1 = wtail[ow][2 * (lane - 2) + 1]; }
        const int off = lane < 2 ? 2 * lane : 4 + 2 * (lane - 2);
        const uint32_t slot = smem_u32(&inbox[par][me][off]);
        const uint32_t bar = smem_u32(&mbar[par]);
        for (int dst = warp; dst < CL; dst += kSvc) st_async_v2(mapa(slot, dst), v0, v1, mapa(bar, dst));
      }
      if (warp == 0) {
        if (MODE & 4) {
          if (lane == 0) while (!try_wait(&mbar[par], (col >> 1) & 1)) {}
          __syncwarp();
        }
        WCand g{0ull, -1, -1.0};
        if (lane < CL) { const double* rs = inbox[par][lane]; g.key = mag_key(fabs(rs[0]) + 1.0); g.idx = (int)__double_as_longlong(rs[2]); }
        WCand best = g;
        if (MODE & 8) {
          best = warp_argmax(g);
          const int o = best.idx > 0 ? (best.idx / 10000) % 16 : 0;
          for (int t = col + lane; t < SMAX; t += 32) U[col % SMAX][t] = inbox[par][o][4 + t];
        }
        if (lane == 0) s_best[par] = best;
        if ((MODE & 64) && lane == 0) s_rcp[par] = __drcp_rn(U[col % SMAX][col % SMAX] + 1.0);
        if ((MODE & 256) && lane == 0 && me == 0) { rec[s * 3] = (double)best.idx; rec[s * 3 + 1] = key_mag(best.key); rec[s * 3 + 2] = best.second; }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (me == 0 && threadIdx.x == 0) { out[MODE == 31 ? 16 : (MODE == 63 ? 17 : (MODE == 127 ? 18 : (MODE == 255 ? 19 : (MODE == 511 ? 20 : MODE))))] = (t1 - t0) / steps; out[31] = s_best[0].key + (long long)s_rcp[0] + (long long)U[1][2] + (long long)cur[0]; }
  cl.sync();
}

static size_t g_dyn = 0;
template <int MODE>
void run(long long* d) {
  auto k = skel<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 20 * 800 * 8;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  static double* rec = nullptr;
  if (!rec) cudaMalloc(&rec, 8 * 3 * 256);
  for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, k, d, 200, rec);
  cudaDeviceSynchronize();
}
int main() {
  long long* d; long long h[32];
  cudaMalloc(&d, sizeof(h)); cudaMemset(d, 0, sizeof(h));
  for (int pass = 0; pass < 1; ++pass) {
  g_dyn = pass ? 200 * 1024 : 0;
  printf("dynamic smem %zu KB\n", g_dyn / 1024);
  run<0>(d); run<1>(d); run<2>(d); run<3>(d); run<4>(d); run<5>(d); run<7>(d); run<12>(d); run<15>(d);
  run<31>(d); run<63>(d); run<127>(d); run<255>(d); run<511>(d);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode 31 (+ row work): %lld cycles/step\n", h[16]);
  printf("mode 63 (+ row work + real tail): %lld cycles/step\n", h[17]);
  printf("mode 127 (+ rcp): %lld, 255 (+ ieee fallback check): %lld, 511 (+ records): %lld cycles/step\n", h[18], h[19], h[20]);
  const int modes[] = {0, 1, 2, 3, 4, 5, 7, 12, 15};
  for (int m : modes) printf("mode %2d (%s%s%s%s): %lld cycles/step\n", m, m & 1 ? "warp-argmax " : "", m & 2 ? "cta-argmax " : "",
                             m & 4 ? "push+wait " : "", m & 8 ? "exchange" : "", h[m]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

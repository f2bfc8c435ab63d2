// Latency of the LUPP warp argmax (redux.sync based) in different CTA states.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct WCand { uint64_t key; int32_t idx; double second; };
__device__ __forceinline__ uint64_t mag_key(double mag) { return static_cast<uint64_t>(__double_as_longlong(mag)) + 1ull; }
__device__ __forceinline__ double key_mag(uint64_t key) { return key ? __longlong_as_double(static_cast<long long>(key - 1ull)) : -1.0; }
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}
__device__ __forceinline__ WCand warp_argmax(const WCand& c) {
  const uint64_t best = warp_max_u64(c.key);
  const int32_t tie_idx = (c.key == best && best != 0) ? c.idx : 0x7fffffff;
  const int32_t widx = __reduce_min_sync(0xffffffffu, tie_idx);
  const bool winner = best != 0 && c.key == best && c.idx == widx;
  const double offer = winner ? c.second : key_mag(c.key);
  const uint64_t okey = offer >= 0.0 ? mag_key(offer) : 0ull;
  const uint64_t sec = warp_max_u64(okey);
  WCand r; r.key = best; r.idx = best ? widx : -1; r.second = key_mag(sec); return r;
}
// mode 0: all warps run the chain; mode 1: only warp 0, others wait at bar.sync;
// mode 2: only warp 0, others spin on FP64 math
__global__ void bench(long long* out, int iters, int mode, double seed) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WCand c{mag_key(seed + lane * 0.37), lane, -1.0};
  long long t0 = clock64();
  if (mode == 0 || warp == 0) {
    for (int i = 0; i < iters; ++i) {
      WCand r = warp_argmax(c);
      c.key = (r.key ^ (uint64_t)lane * 0x9e37u) | 1; c.idx = r.idx + lane; c.second = r.second;
    }
  } else if (mode == 2) {
    double x = seed;
    for (int i = 0; i < iters * 20; ++i) x = fma(x, 1.000001, 1e-9);
    if (x == 12345.0) out[9] = 1;
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) { out[mode] = (t1 - t0) / iters; out[8] = c.key; }
}
__global__ void bench_big(long long* out, int iters, int mode, double seed) {
  extern __shared__ double dyn[];
  dyn[threadIdx.x] = seed;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WCand c{mag_key(dyn[lane] + lane * 0.37), lane, -1.0};
  long long t0 = clock64();
  if (warp == 0) {
    for (int i = 0; i < iters; ++i) {
      WCand r = warp_argmax(c);
      c.key = (r.key ^ (uint64_t)lane * 0x9e37u) | 1; c.idx = r.idx + lane; c.second = r.second;
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[3 + mode] = (t1 - t0) / iters; out[8] = c.key; }
}
__device__ __forceinline__ long long clock_after(unsigned long long dep) {
  long long c;
  asm volatile("{\n.reg .pred p;\nsetp.ne.u64 p, %1, 0x5a5a5a5a5a5a5a5a;\n@p mov.u64 %0, %%clock64;\n@!p mov.u64 %0, %%clock64;\n}\n"
               : "=l"(c) : "l"(dep) : "memory");
  return c;
}
// the LUPP push pattern: compute warps publish WCand to smem, barrier, warp 0 loads and reduces
__global__ void push_pattern(long long* out, int iters, double seed) {
  __shared__ WCand wc[16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long acc_ld = 0, acc_am = 0, acc_bar = 0;
  uint64_t sink = 0;
  for (int it = 0; it < iters; ++it) {
    if (warp >= 4 && lane == 0) wc[warp - 4] = WCand{mag_key(seed + warp * 0.1 + it), warp * 100 + it, 0.5};
    const long long tb = clock64();
    __syncthreads();
    if (warp == 0) {
      const long long t0 = clock_after(tb);
      const WCand c = lane < 12 ? wc[lane] : WCand{0ull, -1, -1.0};
      const long long t1 = clock_after(c.key ^ (uint64_t)c.idx ^ (uint64_t)__double_as_longlong(c.second));
      const WCand r = warp_argmax(c);
      const long long t2 = clock_after(r.key ^ (uint64_t)r.idx);
      acc_ld += t1 - t0; acc_am += t2 - t1; acc_bar += t0 - tb;
      sink ^= r.key;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[6] = acc_bar / iters; out[7] = acc_ld / iters; out[5] = acc_am / iters; out[9] = sink; }
}
int main() {
  long long* d; long long h[10];
  cudaMalloc(&d, sizeof(h));
  for (int m = 0; m < 3; ++m) { bench<<<1, 512>>>(d, 1000, m, 1.5); bench<<<1, 512>>>(d, 1000, m, 1.5); }
  cudaFuncSetAttribute(bench_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024);
  cudaFuncSetAttribute(bench_big, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  bench_big<<<1, 512, 225 * 1024>>>(d, 1000, 0, 1.5);
  bench_big<<<1, 512, 225 * 1024>>>(d, 1000, 0, 1.5);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 225 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, bench_big, d, 1000, 1, 1.5);
  cudaLaunchKernelEx(&cfg, bench_big, d, 1000, 1, 1.5);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("warp_argmax: all warps %lld, warp0 alone (others at barrier) %lld, warp0 + busy warps %lld cycles\n", h[0], h[1], h[2]);
  printf("warp0 alone, 225KB smem: %lld; same in a 16-CTA cluster: %lld (%s)\n", h[3], h[4], cudaGetErrorString(cudaGetLastError()));
  push_pattern<<<1, 512>>>(d, 1000, 1.5);
  push_pattern<<<1, 512>>>(d, 1000, 1.5);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("push pattern: barrier %lld, smem load %lld, warp_argmax %lld cycles (%s)\n", h[6], h[7], h[5], cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Latency (cycles, dependent chains) of the warp-level primitives on the LUPP critical path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}
__device__ __forceinline__ uint64_t warp_max_u64_shfl(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}
__global__ void bench(long long* out, double seed, int iters) {
  const int lane = threadIdx.x & 31;
  long long t0, t1;
  unsigned u = lane * 7919u + (unsigned)seed;
  // 1. redux.sync.max chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) u = __reduce_max_sync(0xffffffffu, u + lane) ^ lane;
  t1 = clock64();
  if (lane == 0) out[0] = (t1 - t0) / iters;
  // 2. shfl chain
  double d = seed + lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = __shfl_sync(0xffffffffu, d, (i + 1) & 31) + 1.0;
  t1 = clock64();
  if (lane == 0) out[1] = (t1 - t0) / iters;
  // 3. warp_max_u64 (redux) chain
  uint64_t k = (uint64_t)u * 0x9e3779b97f4a7c15ull + lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) k = warp_max_u64(k + lane) ^ lane;
  t1 = clock64();
  if (lane == 0) out[2] = (t1 - t0) / iters;
  // 4. warp_max_u64 (shfl butterfly) chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) k = warp_max_u64_shfl(k + lane) ^ lane;
  t1 = clock64();
  if (lane == 0) out[3] = (t1 - t0) / iters;
  // 5. ddiv chain
  double x = seed + lane + 1.5, y = 1.0 + lane * 1e-3;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __ddiv_rn(x, y) + 1.0;
  t1 = clock64();
  if (lane == 0) out[4] = (t1 - t0) / iters;
  // 6. drcp chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = __drcp_rn(y) + 1.0;
  t1 = clock64();
  if (lane == 0) out[5] = (t1 - t0) / iters;
  // 7. Markstein division chain (mul, fma, fma)
  const double r = __drcp_rn(y);
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double q0 = __dmul_rn(x, r);
    const double rr = __fma_rn(-q0, y, x);
    x = __fma_rn(rr, r, q0) + 1.0;
  }
  t1 = clock64();
  if (lane == 0) out[6] = (t1 - t0) / iters;
  // 8. dfma chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __fma_rn(x, 1.0000001, 1e-3);
  t1 = clock64();
  if (lane == 0) out[7] = (t1 - t0) / iters;
  // 9. smem round trip chain
  __shared__ double sm[64];
  sm[lane] = x;
  __syncwarp();
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = ((int)sm[idx] + i) & 31;
  t1 = clock64();
  if (lane == 0) out[8] = (t1 - t0) / iters;
  // 10. __syncthreads with 16 warps
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (lane == 0) out[9] = (t1 - t0) / iters;
  if (lane == 0 && threadIdx.x == 0) out[10] = (long long)(u + k + d + x + y + idx);
}
int main() {
  long long* d;
  long long h[11];
  cudaMalloc(&d, sizeof(h));
  bench<<<1, 512>>>(d, 1.0, 1000);
  bench<<<1, 512>>>(d, 1.0, 1000);
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const char* names[] = {"redux.max chain", "shfl chain", "warp_max_u64 redux", "warp_max_u64 shfl", "ddiv_rn",
                         "drcp_rn", "markstein div", "dfma", "smem load chain", "syncthreads(16 warps)"};
  for (int i = 0; i < 10; ++i) printf("%-24s %lld cycles\n", names[i], h[i]);
  return 0;
}

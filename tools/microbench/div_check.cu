// Exhaustive-ish check that the reciprocal-based division used by the LUPP kernels
//   y = RN(1/b); q = RN(a*y); r = fma(-q, b, a); q' = RN(r*y + q)
// equals IEEE a/b (__ddiv_rn) whenever the guard in lupp.cu admits it (Markstein).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__device__ __forceinline__ double make(uint64_t bits, int mode) {
  // exponent in a moderate range (the guard excludes extremes), random or structured significand
  uint64_t sig = bits & ((1ull << 52) - 1);
  if (mode == 1) sig |= (1ull << 52) - (1ull << (bits >> 58));      // long runs of ones
  if (mode == 2) sig &= ~((1ull << ((bits >> 58) % 52)) - 1);        // trailing zeros
  uint64_t ex = 1023 + (int)((bits >> 52) % 1200) - 600;
  uint64_t sgn = (bits >> 63) << 63;
  return __longlong_as_double((long long)(sgn | (ex << 52) | sig));
}
__device__ __forceinline__ bool guarded(double a, double b, double q) {
  const double aq = fabs(q), aa = fabs(a);
  return aq > 0x1p-968 && aq < 0x1p968 && aa > 0x1p-968 && aa < 0x1p968 && fabs(b) > 0x1p-968 && fabs(b) < 0x1p968;
}
__global__ void check(uint64_t seed, uint64_t n, unsigned long long* bad, unsigned long long* tested) {
  unsigned long long nb = 0, nt = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h1 = mix(seed ^ (2 * i)), h2 = mix(seed ^ (2 * i + 1) ^ 0x9e3779b97f4a7c15ull);
    const int mode = (int)(h1 % 3);
    const double a = make(h1, mode), b = make(h2, (int)(h2 % 3));
    const double y = __drcp_rn(b);
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-q0, b, a);
    const double q = __fma_rn(r, y, q0);
    if (!guarded(a, b, q)) continue;
    ++nt;
    const double ref = __ddiv_rn(a, b);
    if (__double_as_longlong(ref) != __double_as_longlong(q)) ++nb;
  }
  atomicAdd(bad, nb);
  atomicAdd(tested, nt);
}
int main() {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  unsigned long long tb = 0, tt = 0;
  for (int rep = 0; rep < 20; ++rep) {
    cudaMemset(d, 0, 16);
    check<<<148 * 16, 256>>>(0x1234567ull + rep * 0x9e37ull, 1ull << 32, d, d + 1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    tb += h[0]; tt += h[1];
  }
  printf("tested %llu guarded pairs, mismatches vs __ddiv_rn: %llu\n", tt, tb);
  return tb != 0;
}

// Floor of the resident LUPP's fence-free exchange (lupp.cu lupp_resident_kernel): per step every
// CTA publishes a 16-B header (+ optionally a 50-word row tail written by another warp) into a
// fresh, pre-cleared record; warp 0 of every CTA polls all headers (batched), reduces, then polls
// the winner's tail. No LUPP arithmetic. Prints microseconds per step.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;
constexpr uint64_t E = ~0ull;
constexpr int G_MAX = 148, REC = 68, STEPS = 64;

__device__ __forceinline__ void st64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st2(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ uint64_t ld64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ld2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

template <int THREADS>
__global__ void __launch_bounds__(THREADS, 1) xchg(uint64_t* region, int steps, int tail_words, int tail_by_warp1,
                                                     long long* out) {
  __shared__ uint64_t s_key;
  __shared__ int s_win;
  const int g = blockIdx.x, G = gridDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto rec = [&](int s, int q) { return region + (static_cast<size_t>(s) * G_MAX + q) * REC; };
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    // publish: header by warp 0 lane 0, tail by warp 1 (or warp 0)
    const uint64_t key = (static_cast<uint64_t>((g * 7919 + s * 104729) % 1000003) << 20) | g;
    if (warp == 0 && lane == 0) st2(rec(s, g), key, g);
    if (warp == (tail_by_warp1 ? 1 : 0))
      for (int t = lane; t < tail_words; t += 32) st64(rec(s, g) + 4 + t, key + t);
    if (warp == 0) {
      constexpr int QN = (G_MAX + 31) / 32;
      unsigned pend = 0;
      for (int u = 0; u < QN; ++u)
        if (lane + 32 * u < G) pend |= 1u << u;
      uint64_t best = 0;
      int win = 0;
      while (pend) {
        uint64_t k[QN], ix[QN];
#pragma unroll
        for (int u = 0; u < QN; ++u)
          if (pend >> u & 1) ld2(rec(s, lane + 32 * u), k[u], ix[u]);
#pragma unroll
        for (int u = 0; u < QN; ++u)
          if ((pend >> u & 1) && k[u] != E && ix[u] != E) {
            pend &= ~(1u << u);
            if (k[u] > best) best = k[u], win = static_cast<int>(ix[u]);
          }
      }
      for (int o = 16; o; o >>= 1) {
        const uint64_t ob = __shfl_xor_sync(~0u, best, o);
        const int ow = __shfl_xor_sync(~0u, win, o);
        if (ob > best) best = ob, win = ow;
      }
      if (tail_words) {
        const uint64_t* tl = rec(s, win) + 4;
        for (int t = lane; t < tail_words; t += 32)
          while (ld64(tl + t) == E) {
          }
      }
      if (lane == 0) s_key = best, s_win = win;
    }
    __syncthreads();
  }
  if (g == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
  const size_t words = static_cast<size_t>(STEPS) * G_MAX * REC;
  uint64_t* region;
  long long* out;
  cudaMalloc(&region, words * 8);
  cudaMalloc(&out, 8);
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int G = sms < G_MAX ? sms : G_MAX;
  struct Case { int tail, by1; } cases[] = {{0, 0}, {50, 0}, {50, 1}};
  for (auto c : cases) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(region, 0xFF, words * 8);
      int steps = STEPS, tw = c.tail, b1 = c.by1;
      void* args[] = {&region, &steps, &tw, &b1, &out};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((const void*)xchg<736>, G, 736, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      long long cyc;
      cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
      printf("G %d tail %d (by warp %d): %.3f us/step (kernel %.1f us, %lld cycles/step) %s\n", G, tw, b1, ms * 1e3 / steps,
             ms * 1e3, cyc / steps, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

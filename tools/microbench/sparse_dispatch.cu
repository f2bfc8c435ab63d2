// Microbenchmark for the sparse-sign sketch's inner loop (instruction side only, data in
// shared memory): thread = one column of A, NACC sketch-row accumulators in registers, each
// row's 8 (sketch row, sign) targets warp-uniform, dispatched through a switch (jump table).
// Reports elements / clock / SM (HBM parity on B200 needs ~2.8). Also times legacy
// mma.sync s8 (IMMA m16n8k32) throughput for the sliced-integer alternative.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define C2(h) case 2 * (h): if constexpr ((h) < NACC) acc[(h) < NACC ? (h) : 0] += x; break; \
              case 2 * (h) + 1: if constexpr ((h) < NACC) acc[(h) < NACC ? (h) : 0] -= x; break;
#define C8(b) C2(b) C2(b + 1) C2(b + 2) C2(b + 3) C2(b + 4) C2(b + 5) C2(b + 6) C2(b + 7)

template <int NACC>
__device__ __forceinline__ void dispatch(double (&acc)[NACC], uint32_t code, double x) {
  switch (code) {
    C8(0) C8(8) C8(16) C8(24) C8(32) C8(40) C8(48) C8(56)
    default: __builtin_unreachable();
  }
}

#include "sparse_dispatch_brx.inc"
#ifndef KUNROLL
#define KUNROLL 1
#endif
constexpr int kUnroll = KUNROLL;
#ifndef DISPATCH
#define DISPATCH dispatch_brx
#endif

template <int NACC>
__global__ void __launch_bounds__(128, 1) disp_kernel(const uint2* __restrict__ codes, int rows, int reps, double* out) {
  __shared__ double2 tile[32 * 32];   // 64 rows x 32 columns, [col][row pair], xor-swizzled chunks
  __shared__ uint2 cs[64];
  const int lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) tile[q] = make_double2(q * 1e-3, q * 2e-3);
  for (int q = threadIdx.x; q < 64; q += blockDim.x) cs[q] = codes[q];
  __syncthreads();
  double acc[NACC];
#pragma unroll
  for (int h = 0; h < NACC; ++h) acc[h] = 0.0;
  for (int it = 0; it < reps; ++it) {
#pragma unroll 1
    for (int rp = 0; rp < 32; ++rp) {
      const double2 v = tile[lane * 32 + (rp ^ (lane & 7))];
      const uint2 c0 = cs[2 * rp], c1 = cs[2 * rp + 1];
#pragma unroll kUnroll
      for (int k = 0; k < 8; ++k) DISPATCH<NACC>(acc, ((k < 4 ? c0.x : c0.y) >> (8 * (k & 3))) & 0xffu, v.x);
#pragma unroll kUnroll
      for (int k = 0; k < 8; ++k) DISPATCH<NACC>(acc, ((k < 4 ? c1.x : c1.y) >> (8 * (k & 3))) & 0xffu, v.y);
    }
  }
  double s = 0;
#pragma unroll
  for (int h = 0; h < NACC; ++h) s += acc[h];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void imma_kernel(int iters, int* out) {
  int acc[8][4] = {};
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x01010101u, b1 = a0 + 9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int c = 0; c < 8; ++c) for (int v = 0; v < 4; ++v) s += acc[c][v];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
void run_disp(int sms, double clk_ghz) {
  uint2 h[64];
  uint32_t st = 12345;
  for (int r = 0; r < 64; ++r) {
    uint32_t w[2] = {0, 0};
    for (int k = 0; k < 8; ++k) {
      st = st * 1664525u + 1013904223u;
      const uint32_t code = ((st >> 8) % (2 * NACC));
      w[k / 4] |= code << (8 * (k % 4));
    }
    h[r] = make_uint2(w[0], w[1]);
  }
  uint2* d; double* out;
  cudaMalloc(&d, sizeof(h)); cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int wpb : {4}) {
    for (int ctas_per_sm : {1, 2, 4}) {
      const int blocks = sms * ctas_per_sm, reps = 400;
      cudaMalloc(&out, sizeof(double) * blocks * 128);
      disp_kernel<NACC><<<blocks, 32 * wpb>>>(d, 64, 10, out);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      disp_kernel<NACC><<<blocks, 32 * wpb>>>(d, 64, reps, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double elems = double(blocks) * 32 * wpb * reps * 64;  // per thread: 64 rows x 1 column
      const double per_clk_sm = elems / (ms * 1e-3) / (sms * clk_ghz * 1e9);
      printf("dispatch NACC=%d warps/SM=%d: %.3f ms, %.3f elements/clk/SM (= %.0f GB/s of A at %.3f GHz) err=%s\n",
             NACC, wpb * ctas_per_sm, ms, per_clk_sm, elems * 8 / (ms * 1e-3) / 1e9, clk_ghz,
             cudaGetErrorString(cudaGetLastError()));
      cudaFree(out);
    }
  }
  cudaFree(d);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int khz; cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double ghz = khz * 1e-6;
  run_disp<24>(sms, ghz);
  run_disp<56>(sms, ghz);
  {
    int* out; const int blocks = sms * 4, thr = 256, iters = 20000;
    cudaMalloc(&out, sizeof(int) * blocks * thr);
    imma_kernel<<<blocks, thr>>>(10, out);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    imma_kernel<<<blocks, thr>>>(iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(blocks) * (thr / 32) * iters * 8 * 2.0 * 16 * 8 * 32;
    printf("imma m16n8k32 s8: %.3f ms, %.1f TOPS err=%s\n", ms, ops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

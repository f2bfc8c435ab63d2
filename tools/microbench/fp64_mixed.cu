// Do DMMA (mma.sync f64) and DFMA share one FP64 datapath on B200? Warps of one kernel run
// DMMA chains and DFMA chains side by side; total FP64 throughput vs each alone.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mixed(double* out, int iters, int dfma_warps_per_4) {
  const int warp = threadIdx.x >> 5;
  const bool do_dfma = (warp % 4) < dfma_warps_per_4;
  double s = 0;
  if (!do_dfma) {
    double acc[4][4];
    double a[4], b[2];
    for (int v = 0; v < 4; ++v) a[v] = threadIdx.x * 1e-9 + v;
    b[0] = 1.0; b[1] = 0.5;
    for (int c = 0; c < 4; ++c) for (int v = 0; v < 4; ++v) acc[c][v] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
    for (int c = 0; c < 4; ++c) for (int v = 0; v < 4; ++v) s += acc[c][v];
  } else {
    double acc[8];
    const double x = 1.0 + threadIdx.x * 1e-12, y = 0.999999;
    for (int c = 0; c < 8; ++c) acc[c] = c;
    // same flops per iteration as 4 m16n8k8 per warp: 4 * 2048 / 32 lanes = 256 flops = 128 DFMA per lane
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], y, x);
    }
    for (int c = 0; c < 8; ++c) s += acc[c];
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000;
  for (int mode = 0; mode <= 4; ++mode) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    mixed<<<sms * 2, 512>>>(out, 10, mode);
    cudaEventRecord(a);
    mixed<<<sms * 2, 512>>>(out, iters, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warps = sms * 2.0 * 16;
    const double flops = warps * iters * 4 * 2048.0;  // every warp does the same flops
    printf("dfma warps per 4: %d  ->  %.1f TFLOP/s (%s)\n", mode, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

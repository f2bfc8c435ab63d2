// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) shapes vs DFMA.
// Used to pin the FP64 roofline denominator (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_k4(double* out, int iters) {
  double acc[CHAINS][4];
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, b0 = 1.0 + a0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) for (int v = 0; v < 4; ++v) acc[c][v] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) for (int v = 0; v < 4; ++v) s += acc[c][v];
  if (s == 12345.0) out[0] = s;
}
template <int CHAINS>
__global__ void dmma_k8(double* out, int iters) {
  double acc[CHAINS][4];
  double a[4], b[2];
  for (int v = 0; v < 4; ++v) a[v] = threadIdx.x * 1e-9 + v;
  b[0] = 1.0; b[1] = 0.5;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) for (int v = 0; v < 4; ++v) acc[c][v] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) for (int v = 0; v < 4; ++v) s += acc[c][v];
  if (s == 12345.0) out[0] = s;
}
template <int CHAINS>
__global__ void dmma_k16(double* out, int iters) {
  double acc[CHAINS][4];
  double a[8], b[4];
  for (int v = 0; v < 8; ++v) a[v] = threadIdx.x * 1e-9 + v;
  for (int v = 0; v < 4; ++v) b[v] = 1.0 / (v + 1);
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) for (int v = 0; v < 4; ++v) acc[c][v] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) for (int v = 0; v < 4; ++v) s += acc[c][v];
  if (s == 12345.0) out[0] = s;
}
template <int CHAINS>
__global__ void dfma(double* out, int iters) {
  double acc[CHAINS];
  double x = 1.0 + threadIdx.x * 1e-12, y = 0.999999;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], y, x);
  }
  double s = 0; for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[0] = s;
}

template <typename K>
double run(K kern, int blocks, int threads, int iters, double flops_per_warp_iter, const char* name) {
  double* out; cudaMalloc(&out, 8);
  kern<<<blocks, threads>>>(out, 10); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); kern<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double warps = (double)blocks * threads / 32;
  double tf = warps * iters * flops_per_warp_iter / (best * 1e-3) / 1e12;
  printf("%-28s blocks=%d threads=%d  %.3f ms  %.2f TFLOP/s\n", name, blocks, threads, best, tf);
  cudaFree(out);
  return tf;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs=%d clock=%d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  int sm = p.multiProcessorCount, it = 20000;
  for (int tpb : {128, 256, 512}) {
    run(dmma_k4<4>, sm * 2, tpb, it, 4 * 2.0 * 16 * 8 * 4, "dmma m16n8k4 x4chains");
    run(dmma_k4<8>, sm * 2, tpb, it, 8 * 2.0 * 16 * 8 * 4, "dmma m16n8k4 x8chains");
    run(dmma_k8<4>, sm * 2, tpb, it, 4 * 2.0 * 16 * 8 * 8, "dmma m16n8k8 x4chains");
    run(dmma_k16<4>, sm * 2, tpb, it / 2, 4 * 2.0 * 16 * 8 * 16, "dmma m16n8k16 x4chains");
    run(dfma<8>, sm * 2, tpb, it * 4, 8 * 2.0 * 32, "dfma x8chains");
  }
  return 0;
}

// Dependent-chain latency of warp reductions on B200, one warp and 12 warps per SM at once:
// redux.sync (CREDUX) vs shfl.sync (cycles per operation per warp).
#include <cstdio>
#include <cstdint>
__global__ void k(unsigned* out, long long* cyc, int iters) {
  unsigned v = threadIdx.x * 2654435761u;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __reduce_max_sync(0xffffffffu, v ^ i) + threadIdx.x;
  long long t1 = clock64();
  __syncthreads();
  long long t1b = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1 + (i & 15)) + threadIdx.x;
  long long t2 = clock64();
  __syncthreads();
  long long t2b = clock64();
  double d = v;
  for (int i = 0; i < iters; ++i) d = __shfl_xor_sync(0xffffffffu, d, 1 + (i & 15)) + 1.0;
  long long t3 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = v + (unsigned)d;
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1b) / iters; cyc[2] = (t3 - t2b) / iters; }
}
int main() {
  unsigned* o; long long* c; cudaMalloc(&o, 4 * 1024); cudaMalloc(&c, 8 * 4);
  for (int threads : {32, 128, 384, 768}) {
    k<<<1, threads>>>(o, c, 1000); cudaDeviceSynchronize();
    k<<<1, threads>>>(o, c, 1000);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("%4d threads: redux.sync u32 chain %lld cycles/op; shfl.sync u32 %lld; shfl.sync f64 %lld (%s)\n", threads,
           h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

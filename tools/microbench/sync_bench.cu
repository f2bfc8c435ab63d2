// Barrier / exchange latency microbenchmark on B200: grid.sync (cooperative, 148 CTAs),
// cluster.sync (16 CTAs x 1024 threads), __syncthreads, and a DSMEM read round trip.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void grid_sync_kernel(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) { acc += 1.0; g.sync(); }
  if (acc < 0) out[0] = acc;
}
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(1024, 1) cluster_sync_kernel(int iters, double* out) {
  cg::cluster_group c = cg::this_cluster();
  __shared__ double x[32];
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x < 32) x[threadIdx.x] = acc;
    c.sync();
    if (threadIdx.x < 16) acc += *c.map_shared_rank(&x[0], threadIdx.x);
  }
  if (acc < 0) out[0] = acc;
}
__global__ void __launch_bounds__(1024, 1) block_sync_kernel(int iters, double* out) {
  double acc = threadIdx.x;
  for (int i = 0; i < iters; ++i) { acc += 1.0; __syncthreads(); }
  if (acc < 0) out[0] = acc;
}
__global__ void ddiv_kernel(int iters, double* out, double d) {
  double acc = threadIdx.x + 1.0;
  for (int i = 0; i < iters; ++i) acc = __ddiv_rn(acc, d);
  out[threadIdx.x] = acc;
}

int main() {
  double* out; cudaMalloc(&out, 8192);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int iters = 2000;
  for (int blocks : {16, 64, 148}) {
    for (int threads : {256, 1024}) {
      int it = iters; void* args[] = {&it, &out};
      cudaLaunchCooperativeKernel((void*)grid_sync_kernel, blocks, threads, args, 0, 0);
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel((void*)grid_sync_kernel, blocks, threads, args, 0, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("grid.sync     blocks=%3d threads=%4d : %.3f us per sync  (%s)\n", blocks, threads, 1e3 * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  cluster_sync_kernel<<<16, 1024>>>(iters, out);
  cudaEventRecord(e0); cluster_sync_kernel<<<16, 1024>>>(iters, out); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("cluster.sync+DSMEM read  16x1024 : %.3f us per step (%s)\n", 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
  block_sync_kernel<<<1, 1024>>>(iters, out);
  cudaEventRecord(e0); block_sync_kernel<<<1, 1024>>>(iters, out); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("__syncthreads 1024 : %.3f us per sync\n", 1e3 * ms / iters);
  ddiv_kernel<<<1, 32>>>(iters, out, 1.0000001);
  cudaEventRecord(e0); ddiv_kernel<<<1, 32>>>(iters, out, 1.0000001); cudaEventRecord(e1);
  cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("dependent __ddiv_rn : %.1f ns each\n", 1e6 * ms / iters);
  // empty-kernel launch latency
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) block_sync_kernel<<<1, 32>>>(0, out);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("back-to-back tiny kernel: %.2f us per launch\n", 1e3 * ms / 100);
  int it0 = 0; void* args0[] = {&it0, &out};
  cudaEventRecord(e0);
  for (int i = 0; i < 100; ++i) cudaLaunchCooperativeKernel((void*)grid_sync_kernel, 148, 256, args0, 0, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("back-to-back cooperative 148x256 launch: %.2f us per launch\n", 1e3 * ms / 100);
  return 0;
}

// Cost of one cooperative-groups grid barrier (and of a barrier plus a per-step candidate
// exchange through global memory) at the panel-LUPP grid shapes.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void sync_only(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}

__global__ void sync_exchange(int iters, double* cand) {
  cg::grid_group g = cg::this_grid();
  __shared__ double red[8];
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    double r = -1.0;
    for (int q = threadIdx.x; q < gridDim.x; q += blockDim.x) r = fmax(r, cand[(i & 1) * gridDim.x + q]);
    for (int o = 16; o; o >>= 1) r = fmax(r, __shfl_xor_sync(~0u, r, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = red[0];
      for (int w = 1; w < blockDim.x / 32; ++w) m = fmax(m, red[w]);
      acc += m;
      cand[((i + 1) & 1) * gridDim.x + blockIdx.x] = acc + blockIdx.x;
    }
    g.sync();
  }
}

int main() {
  double* cand;
  cudaMalloc(&cand, 8 * 4096);
  cudaMemset(cand, 0, 8 * 4096);
  int grids[] = {16, 74, 148, 196, 296};
  for (int gi = 0; gi < 5; ++gi) {
    int grid = grids[gi], iters = 2000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int kind = 0; kind < 2; ++kind) {
      void* p0[] = {&iters};
      void* p1[] = {&iters, &cand};
      const void* fn = kind ? (const void*)sync_exchange : (const void*)sync_only;
      cudaLaunchCooperativeKernel(fn, grid, 256, kind ? p1 : p0, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, grid, 256, kind ? p1 : p0, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %d %s: %.3f us/step (%s)\n", grid, kind ? "sync+exchange" : "sync", ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

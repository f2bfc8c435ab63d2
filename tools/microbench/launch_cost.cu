// Duration of a near-empty kernel under the launch shapes the engine uses (grid, block,
// dynamic shared memory, cluster dims): separates launch/scheduling cost from work.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void touch(double* out, int n) {
  __shared__ double sm[1];
  if (threadIdx.x == 0) sm[0] = blockIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.z == 0) out[0] = sm[0] + n;
}

static float run(dim3 grid, int threads, size_t smem, int clz, int iters, cudaStream_t st, double* out) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (clz > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = clz;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) cudaLaunchKernelEx(&cfg, touch, out, i);
  // graph of `iters` launches (as the engine replays them)
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < iters; ++i) cudaLaunchKernelEx(&cfg, touch, out, i);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / iters;
}

int main() {
  double* out;
  cudaMalloc(&out, 64);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaFuncSetAttribute(touch, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(touch, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  struct Case { const char* name; dim3 grid; int threads; size_t smem; int clz; };
  Case cases[] = {
      {"gemm1 626x128 73KB cl2", dim3(313, 1, 2), 128, 73728, 2},
      {"gemm1 626x128 73KB nocl", dim3(313, 1, 2), 128, 73728, 1},
      {"gemm1 626x128 0KB cl2", dim3(313, 1, 2), 128, 0, 2},
      {"ub 628x128 52KB cl4", dim3(157, 1, 4), 128, 52224, 4},
      {"ub 628x128 52KB nocl", dim3(157, 1, 4), 128, 52224, 1},
      {"ub 157x128 52KB", dim3(157, 1, 1), 128, 52224, 1},
      {"small 1x32", dim3(1, 1, 1), 32, 0, 1},
      {"lupp 16x768 113KB cl16", dim3(1, 1, 16), 768, 113088, 16},
      {"lupp 16x768 113KB nocl", dim3(1, 1, 16), 768, 113088, 1},
  };
  for (auto& c : cases) printf("%-28s %.2f us/launch\n", c.name, run(c.grid, c.threads, c.smem, c.clz, 200, st, out));
  // alternating shapes (smem carveout changes between consecutive kernels)
  return 0;
}

// Row gathers from a column-major A (the U block's A(I_k,:) at config 4: 50 rows of a 100000 x n
// matrix, every element its own 32-byte sector 800 KB from the next): how fast can HBM serve
// them, and does the thread mapping matter?
//   k1: warp = 32 consecutive columns j, one row q     (32 columns per load instruction)
//   k2: warp = 32 rows q of one column j (rows sorted) (addresses ascending within the column)
//   k3: as k1 with 4 columns per thread in flight
// Output: b x n row-major. Times with CUDA events, the matrix larger than L2.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

__global__ void k1(const double* __restrict__ A, int64_t lda, int64_t n, const int* __restrict__ rows, int b,
                   double* __restrict__ out) {
  const int64_t total = n * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e % n, q = e / n;
    out[q * n + j] = A[rows[q] + j * lda];
  }
}
__global__ void k2(const double* __restrict__ A, int64_t lda, int64_t n, const int* __restrict__ rows, int b,
                   double* __restrict__ out) {
  const int64_t total = n * b;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e % b, j = e / b;
    out[q * n + j] = A[rows[q] + j * lda];
  }
}
__global__ void k3(const double* __restrict__ A, int64_t lda, int64_t n, const int* __restrict__ rows, int b,
                   double* __restrict__ out) {
  const int64_t groups = (n + 127) / 128;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < groups * 32 * b;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lane = e % 32, gq = e / 32, gj = gq % groups, q = gq / groups;
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = gj * 128 + u * 32 + lane;
      v[u] = j < n ? A[rows[q] + j * lda] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t j = gj * 128 + u * 32 + lane;
      if (j < n) out[q * n + j] = v[u];
    }
  }
}

int main(int argc, char** argv) {
  const int64_t m = 100000, n = argc > 1 ? atoll(argv[1]) : 40000;
  const int b = argc > 2 ? atoi(argv[2]) : 50;
  double* A;
  if (cudaMalloc(&A, sizeof(double) * m * n) != cudaSuccess) return 1;
  cudaMemset(A, 0, sizeof(double) * m * n);
  std::mt19937 rng(5);
  std::vector<int> r(b);
  for (auto& x : r) x = static_cast<int>(rng() % m);
  std::sort(r.begin(), r.end());
  int* rows;
  double* out;
  cudaMalloc(&rows, sizeof(int) * b);
  cudaMalloc(&out, sizeof(double) * n * b);
  cudaMemcpy(rows, r.data(), sizeof(int) * b, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto kern, int blocks, int threads) {
    for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(A, m, n, rows, b, out);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int w = 0; w < reps; ++w) {
      cudaMemsetAsync(A + (w % 4) * m * 1000, w, sizeof(double) * m * 1000);  // touch 800 MB: evict L2
      kern<<<blocks, threads>>>(A, m, n, rows, b, out);
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // the same loop without the gathers: the eviction writes alone
    cudaEventRecord(e0);
    for (int w = 0; w < reps; ++w) cudaMemsetAsync(A + (w % 4) * m * 1000, w, sizeof(double) * m * 1000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms0;
    cudaEventElapsedTime(&ms0, e0, e1);
    const double us = (ms - ms0) * 1e3 / reps;
    printf("%s blocks %d threads %d: %.1f us for %d x %lld  (%.1f us scaled to n = 100000; %.0f GB/s of sectors)\n",
           name, blocks, threads, us, b, (long long)n, us * 100000.0 / n, 32.0 * b * n / (us * 1e-6) / 1e9);
  };
  for (int blocks : {148 * 8, 148 * 16, 148 * 64}) {
    run("k1", k1, blocks, 256);
    run("k2", k2, blocks, 256);
    run("k3", k3, blocks, 256);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

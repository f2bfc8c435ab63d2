// DSMEM exchange costs inside a 16-CTA cluster: st.async issue cost and an all-to-all
// "push 32 B + tail to every CTA, wait on own mbarrier" round, as in the LUPP exchange.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void st_async_v2(uint32_t ra, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(ra), "d"(a), "d"(b), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void wait_par(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(par) : "memory");
}

template <int NDST, int NPAIRS>
__global__ void alltoall(long long* out, int iters) {
  __shared__ __align__(16) double inbox[2][16][64];
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int me = cl.block_rank();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  __syncthreads();
  cl.sync();
  long long t_issue = 0, t_total = 0;
  for (int it = 0; it < iters; ++it) {
    const int par = it & 1;
    const long long t0 = clock64();
    if (warp == 0) {
      if (lane == 0) expect_tx(&bar[par], 16 * NPAIRS * 16);  // every CTA receives NPAIRS pairs from each of 16
      // warp 0 pushes to NDST destinations; warps 1.. cover the rest (16 / NDST warps in total)
    }
    if (warp < 16 / NDST && lane < NPAIRS) {
      const uint32_t slot = smem_u32(&inbox[par][me][2 * lane]);
      const uint32_t b = smem_u32(&bar[par]);
      for (int d = warp; d < 16; d += 16 / NDST) st_async_v2(mapa(slot, d), it, lane, mapa(b, d));
    }
    const long long t1 = clock64();
    if (warp == 0) wait_par(&bar[par], (it >> 1) & 1);
    __syncthreads();
    const long long t2 = clock64();
    t_issue += t1 - t0;
    t_total += t2 - t0;
  }
  if (threadIdx.x == 0 && me == 0) { out[0] = t_issue / iters; out[1] = t_total / iters; }
  cl.sync();
}

template <typename K>
void launch(K k, int thr, long long* d) {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16);
  cfg.blockDim = dim3(thr);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, d, 2000);
  cudaDeviceSynchronize();
}
int main() {
  long long* d; long long h[2];
  cudaMalloc(&d, 16);
#define RUN(NDST, NP, THR)                                                                  \
  launch(alltoall<NDST, NP>, THR, d);                                                       \
  launch(alltoall<NDST, NP>, THR, d);                                                       \
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);                                             \
  printf("dst/warp %2d pairs %2d threads %4d: issue %lld cycles, round %lld cycles (%s)\n", NDST, NP, THR, h[0], h[1], \
         cudaGetErrorString(cudaGetLastError()));
  RUN(16, 2, 512) RUN(16, 12, 512) RUN(4, 2, 512) RUN(4, 12, 512) RUN(2, 12, 512) RUN(1, 12, 512) RUN(1, 2, 512)
  RUN(2, 12, 1024) RUN(16, 12, 1024)
  return 0;
}

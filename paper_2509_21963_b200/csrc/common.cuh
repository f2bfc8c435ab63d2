// common.cuh — device helpers shared by every IterativeCUR kernel (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "crmath.cuh"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_2509_21963_b200 kernels target sm_100a only"
#endif

namespace itercur_b200 {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------------
// Philox4x32-10 keyed exactly like proj/src/rng.cpp:20-52 (counter_for / to_unit /
// normal_at). Integer and to_unit parts are bit-exact; log/cos are correctly rounded
// (crmath.cuh) — the reference's glibc is not, on ~0.2% of inputs.
// ---------------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 ctr, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * ctr.x;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * ctr.z;
    ctr = U4{static_cast<uint32_t>(p1 >> 32) ^ ctr.y ^ k0, static_cast<uint32_t>(p1),
             static_cast<uint32_t>(p0 >> 32) ^ ctr.w ^ k1, static_cast<uint32_t>(p0)};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return ctr;
}

__host__ __device__ __forceinline__ U4 counter_for(uint32_t stream, int64_t i, int64_t j) {
  return U4{stream, static_cast<uint32_t>(i), static_cast<uint32_t>(j),
            static_cast<uint32_t>((static_cast<uint64_t>(i) >> 32) ^ ((static_cast<uint64_t>(j) >> 32) << 8))};
}

__host__ __device__ __forceinline__ double to_unit(uint32_t hi, uint32_t lo) {
  const uint64_t bits = (static_cast<uint64_t>(hi) << 32) | lo;
  return (static_cast<double>(bits >> 11) + 0.5) * 0x1p-53;
}

__device__ __forceinline__ double normal_at_dev(uint64_t seed, uint32_t stream, int64_t i, int64_t j) {
  const U4 r = philox4x32_10(counter_for(stream, i, j), static_cast<uint32_t>(seed),
                             static_cast<uint32_t>(seed >> 32));
  // sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2), rounding order of rng.cpp:51, with
  // correctly rounded log / cos (crmath.cuh) so the stream matches glibc wherever glibc
  // itself rounds correctly.
  return crm::box_muller_cos(to_unit(r.x, r.y), to_unit(r.z, r.w));
}

__device__ __forceinline__ double uniform_at_dev(uint64_t seed, uint32_t stream, int64_t i, int64_t j) {
  const U4 r = philox4x32_10(counter_for(stream, i, j), static_cast<uint32_t>(seed),
                             static_cast<uint32_t>(seed >> 32));
  return to_unit(r.x, r.y);
}

// ---------------------------------------------------------------------------------
// Deterministic (value, lowest-index) pivot candidates: proj/src/select.cpp:40-48 scans
// ascending with a strict '>' so ties go to the lowest index. `second` tracks the
// runner-up magnitude for the parity checker's margin log.
// ---------------------------------------------------------------------------------
// a / p correctly rounded from a precomputed y = RN(1/p) (Markstein: q0 = RN(a y), r = a - q0 p
// exactly, q = RN(q0 + r y)); outside the exponent range where the theorem holds (or for a = 0)
// the IEEE division itself. p_ok: |p| inside [2^-968, 2^968].
static __device__ __noinline__ double ieee_div(double a, double p) { return __ddiv_rn(a, p); }
__device__ __forceinline__ double div_by_pivot(double a, double p, double y, bool p_ok) {
  const double q0 = __dmul_rn(a, y);
  const double r = __fma_rn(-q0, p, a);
  const double q = __fma_rn(r, y, q0);
  const double aq = fabs(q), aa = fabs(a);
  if (p_ok && aq > 0x1p-968 && aq < 0x1p968 && aa > 0x1p-968 && aa < 0x1p968) return q;
  return ieee_div(a, p);
}
__device__ __forceinline__ bool pivot_in_range(double p) { return fabs(p) > 0x1p-968 && fabs(p) < 0x1p968; }

struct Cand {
  double mag;
  double second;
  int64_t idx;
};
__device__ __forceinline__ Cand cand_empty() { return Cand{-1.0, -1.0, -1}; }
__device__ __forceinline__ bool cand_beats(double am, int64_t ai, double bm, int64_t bi) {
  return am > bm || (am == bm && ai >= 0 && (bi < 0 || ai < bi));
}
__device__ __forceinline__ Cand cand_merge(const Cand& a, const Cand& b) {
  if (cand_beats(a.mag, a.idx, b.mag, b.idx)) return Cand{a.mag, fmax(a.second, b.mag), a.idx};
  return Cand{b.mag, fmax(b.second, a.mag), b.idx};
}
__device__ __forceinline__ Cand cand_shfl_down(const Cand& c, int off) {
  Cand o;
  o.mag = __shfl_down_sync(0xffffffffu, c.mag, off);
  o.second = __shfl_down_sync(0xffffffffu, c.second, off);
  o.idx = __shfl_down_sync(0xffffffffu, c.idx, off);
  return o;
}
__device__ __forceinline__ Cand warp_reduce_cand(Cand c) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) c = cand_merge(c, cand_shfl_down(c, off));
  return c;  // lane 0 holds the result (merge is associative & commutative on the key)
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  return v;
}

// Block-wide deterministic sum (fixed tree); result valid in thread 0.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* smem_scratch) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) smem_scratch[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) t += smem_scratch[w];
  }
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------------
// FP64 tensor-core MMA (DMMA): sm_100 has no tcgen05 f64 kind, so the f64
// tensor path is the warp-level mma.sync m16n8k8. Fragment layout (CuTe SM90 traits):
//   a[v0 + 2 v1] = A(g + 8 v0, t + 4 v1), b[v] = B(t + 4 v, g), c[v0 + 2 v1] = C(g + 8 v1, 2t + v0)
// with g = lane / 4, t = lane % 4. Kernels permute K so logical (t, t+4) = physical
// (2t, 2t+1): one 16-byte shared load per fragment pair.
// ---------------------------------------------------------------------------------
// programmatic dependent launch: wait for the preceding kernel's completion and memory
// (no-op when launched without the PDL attribute); allow the next kernel to launch early
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
#ifdef ITERCUR_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}

__device__ __forceinline__ void dmma_16x8x8(double (&d)[4], double a0, double a1, double a2, double a3, double b0,
                                            double b1) {
  asm(  // not volatile: lets the scheduler interleave independent MMAs with loads
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

// ---------------------------------------------------------------------------------
// mbarrier + TMA (cp.async.bulk.tensor) helpers
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// The retry loops are C++ loops around a single try_wait: a branch inside inline asm is
// invisible to the compiler's reconvergence analysis, and lanes leaving such a loop at
// different times stay diverged afterwards (every later warp collective then takes the
// slow divergent path).
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// Byte offset of element (row, k) inside a [rows][16 doubles] tile written by TMA with
// CU_TENSOR_MAP_SWIZZLE_128B (16-byte chunk index XOR row % 8; tile base 1024-B aligned).
__device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t k) {
  return row * 128u + ((((k >> 1) ^ (row & 7u)) & 7u) << 4) + ((k & 1u) << 3);
}

}  // namespace itercur_b200

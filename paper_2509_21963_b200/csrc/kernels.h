// kernels.h — host-side launchers of the sm_100a IterativeCUR kernels (internal API).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <utility>

namespace itercur_b200 {

// A/B and tuning switches: set, non-empty and not "0"
inline bool env_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] && !(e[0] == '0' && e[1] == 0);
}

constexpr uint32_t kStreamSketch = 1;      // RngStream::Sketch, proj/include/itercur/rng.hpp:13
constexpr uint32_t kStreamSluppSketch = 2; // RngStream::SluppSketch (the s-LUPP baseline, baselines.cpp:44-46)
constexpr uint32_t kStreamSparseSign = 7;  // new tag
constexpr int kSketchGaussian = 0;
constexpr int kSketchSparseSign = 1;

__host__ __device__ inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
__host__ __device__ inline int64_t ceil_div(int64_t x, int64_t a) { return (x + a - 1) / a; }

// Programmatic dependent launch for the per-iteration kernel chain: while the engine enqueues
// an iteration batch (pdl_scope), launches carry cudaLaunchAttributeProgrammaticStream-
// Serialization, so each kernel is launched while its predecessor drains; every such kernel
// calls griddep_wait() (common.cuh) before touching its predecessor's output.
bool pdl_enabled();
struct PdlScope {
  bool prev;
  explicit PdlScope(bool on);
  ~PdlScope();
};
// cudaLaunchKernelEx with optional cluster dims (cluster.x == 0: no cluster attribute) and the
// PDL attribute when enabled.
template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, dim3 cluster,
                      Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (cluster.x > 0) {  // explicit cluster launch (dim3(0, ...) = none)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster.x;
    attr[na].val.clusterDim.y = cluster.y;
    attr[na].val.clusterDim.z = cluster.z;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------- sketch
// Dense sketch operator S (rows_pad x ldg, row-major: S[h * ldg + k]), rows h >= c and
// columns k >= m are zero. Gaussian: S(h,k) = normal_at(seed, Sketch, h, k)
// (proj/src/sketch.cpp:19 -> rng.cpp:61-67). Sparse-sign: +-1 at the A.8 positions.
cudaError_t launch_gen_sketch_operator(double* S, int64_t rows_pad, int64_t ldg, int64_t c, int64_t m, uint64_t seed,
                                       int kind, int zeta, cudaStream_t st, uint32_t stream_tag = kStreamSketch);

struct SketchStats {
  double* d_asq;  // ||A||_F^2 (device scalar)
  double* d_ysq;  // ||Y||_F^2 (device scalar)
};

// Y (c_pad x n, ld c_pad, column-major) = scale * S(0:c_pad, :) * A, plus ||A||^2 and ||Y||^2
// reduced deterministically into device scalars. Uses TMA when A's layout allows it.
// Returns the split count and timing info via out params (host side).
struct SketchLaunchInfo {
  int splits = 1;
  int ctas = 0;
  int nt = 0;
  bool tma = false;
  int dominant_launches = 0;  // launches of the DMMA kernel
};
cudaError_t run_sketch_apply(const double* A, int64_t m, int64_t n, int64_t lda, const double* S, int64_t ldg,
                             int64_t c_pad, double scale, double* Y, double* workspace, int64_t workspace_elems,
                             const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info);
int64_t sketch_workspace_elems(int64_t m, int64_t n, int64_t c_pad);
// Sparse-sign sketch as a sparse operator (no dense Omega): Y (c_pad x n, ld c_pad) =
// scale * Omega * A generated from (seed, c, zeta) on the fly, ||A||^2 and ||Y||^2 as above.
bool sparse_sketch_supported(int64_t c, int zeta);
int64_t sparse_sketch_workspace_elems(int64_t m, int64_t n, int64_t c_pad, int zeta);
cudaError_t run_sketch_apply_sparse(const double* A, int64_t m, int64_t n, int64_t lda, uint64_t seed, int64_t c,
                                    int64_t c_pad, int zeta, double scale, double* Y, double* ws, int64_t ws_elems,
                                    const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info);
// Sparse-sign sketch on the integer tensor path (56-bit fixed-point slices of A x int8 operator,
// mma.sync s8; sketch.cu). Needs c_pad <= 64, even lda and a 16-byte aligned A.
bool sparse_sketch_imma_supported(const double* A, int64_t lda, int64_t c_pad);
int64_t sparse_sketch_imma_workspace_elems(int64_t m, int64_t n, int64_t c_pad);
cudaError_t run_sketch_apply_sparse_imma(const double* A, int64_t m, int64_t n, int64_t lda, uint64_t seed, int64_t c,
                                         int64_t c_pad, int zeta, double scale, double* Y, double* ws, int64_t ws_elems,
                                         const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info,
                                         bool operator_ready, bool kernel_only = false);
// The same on tcgen05 (kind::i8, TMEM accumulators; TMA-staged A tiles): c_pad <= 64.
bool sparse_sketch_umma_supported(const double* A, int64_t m, int64_t n, int64_t lda, int64_t c_pad);
int64_t sparse_sketch_umma_workspace_elems(int64_t m, int64_t n, int64_t c_pad);
cudaError_t run_sketch_apply_sparse_umma(const double* A, int64_t m, int64_t n, int64_t lda, uint64_t seed, int64_t c,
                                         int64_t c_pad, int zeta, double scale, double* Y, double* ws, int64_t ws_elems,
                                         const SketchStats& stats, cudaStream_t st, SketchLaunchInfo* info,
                                         bool operator_ready, bool kernel_only = false);
// Stand-alone timing hook: the DMMA kernel only (for roofline measurement).
cudaError_t run_sketch_dmma_only(const double* A, int64_t m, int64_t n, int64_t lda, const double* S, int64_t ldg,
                                 int64_t c_pad, double* Y, double* workspace, int64_t workspace_elems, cudaStream_t st,
                                 SketchLaunchInfo* info);

// ------------------------------------------------------------------------------ LUPP
struct LuppArgs {
  double* W;                // rows x cols_max column-major working copy (modified in place)
  int64_t rows;
  int64_t ldw;
  int cols_max;             // columns present in W
  const int* d_steps;       // dynamic requested steps (device int), capped by cols_max
  uint8_t* mask;            // per-row ban mask: 1 = permanently banned, `epoch` = banned in this call
  uint8_t epoch;
  const double* d_norm_sq;  // ||M||_F^2 for the absolute floor; nullptr -> computed from W
  double pivot_floor;
  int64_t* d_idx;           // out: pivots
  double* d_best;           // out: |pivot|
  double* d_second;         // out: runner-up magnitude (margin log)
  int* d_count;             // out: accepted pivots
  int* d_width_out = nullptr;        // optional out: min(count, *d_width_cap)
  const int* d_width_cap = nullptr;
  int requested_b;          // for `truncated` semantics (host side)
  // slot-tag generation for the tagged exchange: when d_gen_k is set the generation is
  // derived on the device, gen_base | (k << 1) | gen_which, so captured graphs replay safely
  const int64_t* d_gen_k = nullptr;
  uint32_t gen_base = 0;
  int gen_which = 0;
  // optional (cluster path): emit the LU factors of the pivot rows, row s of the block =
  // (multipliers of steps < s, eliminated entries from column s on) — exactly the
  // factorisation of W(I, 0:count) in pivot order; written at lu_out + (*d_lu_r) * lu_ld
  double* lu_out = nullptr;
  int64_t lu_ld = 0;
  const int64_t* d_lu_r = nullptr;
  // optional (cluster path, see lupp_fuses_iteration_work): the iteration-begin bookkeeping of
  // misc.cu iter_begin_kernel runs in the prologue (steps then come from the loop control, not
  // d_steps) ...
  void* begin_ctl = nullptr;   // IterCtl*
  void* begin_slot = nullptr;  // IterState*
  // ... and up to two gathers indexed by the pivots just chosen run after the last step:
  // out[k + q*ldo] = src[k*row_stride + idx[q]*col_stride] for k < K, q < count, zero for
  // count <= q < w_fill; K = min(kmax, *k_cap) when k_cap is set.
  struct Gather {
    const double* src = nullptr;
    int64_t row_stride = 0, col_stride = 0, kmax = 0;
    const int64_t* k_cap = nullptr;
    double* out = nullptr;
    int64_t ldo = 0;
    int w_fill = 0;
  } post[2];
};
// QRCP selection (qrcp.cu, select.cpp:79-117): candidates are the ncand vectors of length len
// at W[i*rs + j*cs] (modified in place); same outputs as the LUPP launchers.
struct IterCtl;
size_t qrcp_scratch_bytes();
cudaError_t run_qrcp(double* W, int64_t ncand, int len, const int* d_len, int64_t rs, int64_t cs, const int* d_steps,
                     int steps_max,
                     uint8_t* mask, uint8_t epoch, const double* d_norm_sq, double pivot_floor, int64_t* d_idx,
                     double* d_best, double* d_second, int* d_count, int* d_width_out, const int* d_width_cap,
                     void* scratch, const IterCtl* ctl, cudaStream_t st);
// true when run_lupp_with_scratch takes the cluster path for these arguments (which honours
// begin_ctl / post gathers; the other paths ignore them and the caller launches them itself)
bool lupp_fuses_iteration_work(const LuppArgs& a);
size_t lupp_scratch_bytes(int b);
cudaError_t lupp_scratch_init(void* scratch, cudaStream_t st);  // after every allocation
// column-sharded engine building blocks (shard.cu)
cudaError_t launch_lupp_dist_step(double* W, int64_t rows, int64_t ldw, int steps, int s, const double* P,
                                  int64_t piv_local, uint8_t* live, int64_t row_offset, double* cand,
                                  cudaStream_t st);
cudaError_t launch_dense_lu(double* D, int w, int64_t ldd, cudaStream_t st);
cudaError_t run_lupp_with_scratch(const LuppArgs& a, void* scratch, cudaStream_t st, int* grid_used);
cudaError_t launch_clear_epochs(uint8_t* mask, int64_t count, cudaStream_t st);
// benchmarking: 0 automatic, 1 cluster only, 2 grid shared-memory only, 3 global only
void set_lupp_force_path(int path);
void set_lupp_debug_trace(long long* dbg);  // per-step clock64() trace of CTA 0 (grid path)
void set_lupp_grid_trace(long long* gdbg);  // resident path: globaltimer stamps of every CTA per step

// one kernel per translation unit (module): itercur_preload loads every function of each module
const void* module_anchor_gemm();
const void* module_anchor_lupp();
const void* module_anchor_misc();
const void* module_anchor_qrcp();
const void* module_anchor_shard();
const void* module_anchor_sketch();

}  // namespace itercur_b200

// engine.cu — the C++ host driver of the B200 IterativeCUR engine and its C-ABI
// (include/itercur_b200.h). It restates the loop of itercur::iterative_cur
// (proj/src/driver.cpp:48-167) over device-resident state, in the incremental block-LU
// (Schur) form of SURVEY.md A.7:
//
//   sketch    Y = S*A once (DMMA + TMA), ||A||, ||Y||                 sketch.cu
//   loop k:   J_k  = LUPP(Y^T)                                        lupp.cu
//             S_row = A(:,J_k) - L * Rt(:,J_k)   -> L_k                gemm.cu
//             I_k  = LUPP(S_row)                                      lupp.cu
//             D_k^{-1} from S_row(I_k, :)                             misc.cu
//             U_k^T = A(I_k,:)^T - Rt^T * L(I_k,:)^T ; Rt_k = D_k^{-1} U_k   gemm.cu
//             Y   -= Y(:,J_k) * Rt_k  (in place, ||Y||^2 fused)       gemm.cu
//             rho = ||Y|| / ||S*A||  -> one 64-B+ D2H read per iteration
//
// so CUR = L * Rt with C = A(:,J), R = A(I,:), core = A(I,J)^{-1} = (L(I,:) Rt(:,J))^{-1}
// exported on demand. A is never re-read after the sketch except through the gathered
// columns / rows of the selected blocks.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/itercur_b200.h"
#include "collectives.h"
#include "gemm.h"
#include "kernels.h"
#include "misc.h"

using namespace itercur_b200;

namespace {

// ------------------------------------------------------------------ errors
struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg) { throw ApiError(code, msg); }
void ck(cudaError_t e, const char* what, int line) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation)
      fail(ITERCUR_E_OOM, std::string("device allocation failed (") + what + ")");
    fail(ITERCUR_E_CUDA, std::string("CUDA error '") + cudaGetErrorString(e) + "' at engine.cu:" +
                             std::to_string(line) + " (" + what + ")");
  }
}
#define CK(x) ck((x), #x, __LINE__)

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ITERCUR_OK;
  } catch (const ApiError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return ITERCUR_E_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ITERCUR_E_RUNTIME;
  }
}

// ------------------------------------------------------------------ device buffers
// Stream-ordered allocations from the device's default memory pool (release threshold
// raised once), so the per-run workspaces cost no cudaMalloc / cudaFree synchronisation
// after the first run.
thread_local cudaStream_t g_alloc_stream = nullptr;

// The engine's own non-blocking work stream (one per host thread, never destroyed): the
// iteration batches are captured into CUDA graphs, which the legacy default stream cannot do.
// Streams are cached per host thread AND per device ordinal: a thread that runs on cuda:0 and
// later on cuda:1 must not launch into (or allocate on) a stream of the first device.
constexpr int kMaxDevices = 64;
int current_device() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) fail(ITERCUR_E_CUDA, "device ordinal out of range");
  return dev;
}
cudaStream_t work_stream() {
  thread_local cudaStream_t s[kMaxDevices] = {};
  const int dev = current_device();
  if (!s[dev]) CK(cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking));
  return s[dev];
}

// A second work stream for graph branches off the iteration's critical path, with its two events.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream() {
  thread_local SideStream ss[kMaxDevices];
  SideStream& x = ss[current_device()];
  if (!x.s) {
    CK(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&x.join, cudaEventDisableTiming));
  }
  return x;
}

void configure_mempool_once() {
  static std::atomic<bool> done[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return;
  if (done[dev].load()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev].store(true);
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    count = 0;
  }
  void alloc(size_t n) {
    reset();
    if (n == 0) n = 1;
    st = g_alloc_stream;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(T), st));
    count = n;
  }
  void swap(DevBuf& o) {
    std::swap(p, o.p);
    std::swap(count, o.count);
    std::swap(st, o.st);
  }
};

struct Events {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t get(size_t i) {
    while (ev.size() <= i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev.push_back(e);
    }
    return ev[i];
  }
  ~Events() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, a, b));
  return 1e-3 * ms;
}

}  // namespace

// ====================================================================== the run handle
// Column-sharded runs: A is split by columns into contiguous shards. A process
// computes `nloc` of them: one (NCCL mode: one process per GPU, `world` ranks in `comm`) or all
// of them on one device (emulation: every shard's kernels run on their own column range, the
// collectives become the equivalent device copies). Replicated state (L, D_k, masks, I, J, the
// loop control, Wc = Y^T(:, 0:b)) is identical everywhere; per-shard state (A, Y, R~) covers the
// shard's columns only.
struct ShardSpec {
  bool active = false;
  int nloc = 1;
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  int64_t n_total = 0;             // global column count
  std::vector<int64_t> goff, cnt;  // local shards: global column offset and count
  bool emulated() const { return active && comm == nullptr; }
};

struct itercur_run {
  int device = 0;
  cudaStream_t stream = nullptr;   // the caller's stream (accessors run on it)
  cudaStream_t wstream = nullptr;  // the engine's work stream for iterative_cur (capturable)
  int64_t m = 0, n = 0, lda = 0;
  const double* A = nullptr;
  DevBuf<double> A_owned;  // host entry: device copy of A (freed when the call returns unless kept)
  DevBuf<double> Cg, RgT;  // host entry without the copy: C = A(:,J) (m x r), R^T = A(I,:)^T (n x r)
  itercur_config cfg{};
  int64_t c = 0, cp = 0;
  int64_t r = 0;
  std::vector<int64_t> I, J;
  std::vector<int64_t> block_start, block_width;
  int32_t status = ITERCUR_CONVERGED;
  double final_rho = 1.0, threshold = 0.0, sketch_s = 0.0, total_s = 0.0, ga_norm = 0.0, a_norm = 0.0;
  std::string note;
  std::vector<itercur_iteration_record> iters;
  std::vector<int32_t> step_kind;
  std::vector<int64_t> step_iter, step_index;
  std::vector<double> step_best, step_second;
  // factors (incremental block-LU form)
  DevBuf<double> L;     // m x capL, column-major, ld ldL
  DevBuf<double> Rt;    // capL rows of n, row-major (Rt[q * ldR + j])
  DevBuf<double> Dinv;  // per block: LU of D_k (w x w, ld bmax) at offset start * bmax
  DevBuf<int> Piv;      // QRCP rows only: D_k's partial-pivoting permutation at offset start
  DevBuf<int64_t> dI, dJ;
  int64_t ldL = 0, ldR = 0, capL = 0, bmax = 0;
  int64_t launches = 0;  // kernels of this library launched by the run (sketch + loop)
  ShardSpec sh;          // column sharding (inactive: the plain single-device run)
};

namespace {

int64_t even(int64_t x) { return x + (x & 1); }
// The column partition of sharded runs: contiguous blocks of an even width (16-byte aligned
// offsets), rank r owning [r * blk, min((r + 1) * blk, n)).
int64_t shard_block(int64_t n, int world) { return round_up(ceil_div(n, world), 2); }

// StoppingConfig defaults, proj/include/itercur/driver.hpp:18-26; SelectionMethod select.hpp:12-15
itercur_config default_config() {
  itercur_config c{};
  c.epsilon = 1e-6;
  c.b = 50;
  c.delta = 0.0;
  c.alpha = 0.05;
  c.risk_adjust = 0;
  c.max_rank = 0;
  c.max_iters = 0;
  c.col_method = ITERCUR_PIVOT_LUPP;
  c.row_method = ITERCUR_PIVOT_LUPP;
  c.pivot_floor = 1e-13;
  c.row_pivot_floor = 1e-13;
  c.observer = nullptr;
  c.observer_user = nullptr;
  c.keep_device_copy = 0;
  c.seed = 0;
  c.sketch_kind = ITERCUR_SKETCH_GAUSSIAN;
  c.sparse_nnz = 8;
  c.profile = 0;
  return c;
}

// adjusted_threshold, proj/src/driver.cpp:28-39
double adjusted_threshold_impl(double epsilon, double delta, double alpha, int64_t c) {
  if (!(alpha > 0.0 && alpha < 1.0)) fail(ITERCUR_E_INVALID_ARGUMENT, "alpha must lie in (0, 1)");
  if (delta < 0.0) fail(ITERCUR_E_INVALID_ARGUMENT, "delta must be nonnegative");
  if (c < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "sketch rows must be positive");
  const double nla = -std::log(alpha);
  if (static_cast<double>(c) <= 4.0 * nla) fail(ITERCUR_E_DOMAIN, "block too small for requested alpha");
  const double xi = (1.0 + delta) * std::sqrt(1.0 - 2.0 * std::sqrt(nla / static_cast<double>(c)));
  return xi * epsilon;
}
// gratton_tail, proj/src/driver.cpp:41-46
double gratton_tail_impl(int64_t c, double tau) {
  if (c < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "sketch rows must be positive");
  if (!(tau > 1.0)) fail(ITERCUR_E_DOMAIN, "tau must exceed 1");
  const double t2 = tau * tau;
  return std::exp(-static_cast<double>(c) * (t2 - 1.0) * (t2 - 1.0) / (4.0 * t2 * t2));
}

int64_t sketch_rows(int64_t b) { return (11 * b) / 10; }  // proj/include/itercur/sketch.hpp:10

void check_method(int32_t kind) {
  if (kind == ITERCUR_PIVOT_OSINSKY) fail(ITERCUR_E_RUNTIME, "Osinsky selection not implemented");
  if (kind != ITERCUR_PIVOT_LUPP && kind != ITERCUR_PIVOT_QRCP) fail(ITERCUR_E_LOGIC, "unknown selection method");
}

// ||A||_F^2 via a dedicated pass (only used when validation must report in the reference's
// order before the fused sketch pass runs, and for the true-error denominator).
double device_sumsq(const double* x, int64_t rows, int64_t cols, int64_t ld, cudaStream_t st) {
  DevBuf<double> part, out;
  part.alloc(148 * 8);
  out.alloc(1);
  CK(launch_sumsq(x, rows, cols, ld, part.p, 148 * 8, out.p, st));
  double h = 0.0;
  CK(cudaMemcpyAsync(&h, out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h;
}

// ---- the sketch apply (make_sketch, sketch.cpp:10-24), shared by the run and the stage entries.
// Sparse-sign operator, four kernels (ITERCUR_SPARSE_SKETCH selects; default: 3 when c_pad > 32,
// else 2 — the faster one at each shape on B200, tools/sketch_modes.py):
//   3  tcgen05 kind::i8 (sketch.cu sparse_sketch_umma_kernel): A as int8 slices of a per-column
//      fixed-point form, written by the converter warps straight into TMEM as the MMA's A operand,
//      int32 accumulators in TMEM, TMA-staged A tiles, persistent CTAs: 83-88% of HBM at c = 55;
//   2  the same contraction on mma.sync s8 (register accumulators): 83% of HBM at c_pad = 24 (the
//      tcgen05 form: 79%, equal full-run time at config 2; tcgen05 is the default at every c_pad);
//   0  FP64 DMMA over the materialised +-1 operator (FP64-bound once c_pad > ~24: 37% at c = 55);
//   1  the sparse list walk (bitwise equal to the oracle's sparse loop; bound by shared-memory
//      reads of every (row, target) pair: 3.9 ms vs DMMA 2.7 ms at 40000 x 20000, c = 55).
struct SketchBuffers {
  DevBuf<double> S, ws;
};
enum SparseMode { kSparseDense = 0, kSparseList = 1, kSparseImma = 2, kSparseUmma = 3 };
static int sparse_sketch_mode(int kind, int64_t c, int64_t cp, int zeta_eff, const double* A, int64_t lda) {
  if (kind != kSketchSparseSign) return kSparseDense;
  const char* e = getenv("ITERCUR_SPARSE_SKETCH");
  const int want = (e && e[0]) ? atoi(e) : kSparseUmma;  // tcgen05 kind::i8 at every c_pad it supports
  if (want == kSparseList && sparse_sketch_supported(c, zeta_eff)) return kSparseList;
  if (want == kSparseUmma && sparse_sketch_umma_supported(A, 0, 0, lda, cp)) return kSparseUmma;
  if ((want == kSparseImma || want == kSparseUmma) && sparse_sketch_imma_supported(A, lda, cp)) return kSparseImma;
  return kSparseDense;
}
static int zeta_effective(int kind, int sparse_nnz, int64_t c) {
  return kind == kSketchSparseSign ? static_cast<int>(std::min<int64_t>(std::max(sparse_nnz, 1), c)) : 0;
}
// The sparse-sign nonzeros per column: the oracle rejects zeta < 1 (itercur_oracle.cpp make_sketch);
// the device kernels draw at most kMaxSparseNnz = 16 slots per column into fixed-size per-thread
// arrays (sketch.cu sparse_sign_slots), so min(zeta, c) above 16 is rejected rather than overrun.
constexpr int kMaxSparseNnz = 16;
static void check_sparse_nnz(int kind, int sparse_nnz, int64_t c) {
  if (kind != kSketchSparseSign) return;
  if (sparse_nnz < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "sparse_nnz must be at least 1");
  if (std::min<int64_t>(sparse_nnz, c) > kMaxSparseNnz)
    fail(ITERCUR_E_INVALID_ARGUMENT, "sparse_nnz above 16 is not supported by the B200 engine");
}
// Y (cp x n, ld cp) = scale * S * A, ||A||^2 -> stats.d_asq, ||Y||^2 -> stats.d_ysq. Returns the
// number of kernel launches.
static int apply_sketch(const double* A, int64_t m, int64_t n, int64_t lda, int kind, int sparse_nnz, uint64_t seed,
                        uint32_t stream_tag, int64_t c, int64_t cp, double* Y, const SketchStats& stats,
                        SketchBuffers& buf, cudaStream_t st, SketchLaunchInfo* info = nullptr,
                        bool operator_ready = false) {
  check_sparse_nnz(kind, sparse_nnz, c);
  const int ze = zeta_effective(kind, sparse_nnz, c);
  const double scale = kind == kSketchSparseSign ? 1.0 / std::sqrt(static_cast<double>(ze)) : 1.0;
  const int mode = sparse_sketch_mode(kind, c, cp, ze, A, lda);
  if (mode == kSparseList) {
    const int64_t wse = sparse_sketch_workspace_elems(m, n, cp, ze);
    if (buf.ws.count < static_cast<size_t>(wse)) buf.ws.alloc(wse);
    CK(run_sketch_apply_sparse(A, m, n, lda, seed, c, cp, ze, scale, Y, buf.ws.p, wse, stats, st, info));
    return 4;
  }
  if (mode == kSparseUmma) {
    const int64_t wse = sparse_sketch_umma_workspace_elems(m, n, cp);
    if (buf.ws.count < static_cast<size_t>(wse)) buf.ws.alloc(wse);
    CK(run_sketch_apply_sparse_umma(A, m, n, lda, seed, c, cp, ze, scale, Y, buf.ws.p, wse, stats, st, info, false));
    return 6;
  }
  if (mode == kSparseImma) {
    // the int8 operator lives in the workspace; it is regenerated per call (m threads)
    const int64_t wse = sparse_sketch_imma_workspace_elems(m, n, cp);
    if (buf.ws.count < static_cast<size_t>(wse)) buf.ws.alloc(wse);
    CK(run_sketch_apply_sparse_imma(A, m, n, lda, seed, c, cp, ze, scale, Y, buf.ws.p, wse, stats, st, info, false));
    return 6;
  }
  const int64_t ldg = round_up(m, 32);
  int launches = 0;
  if (!operator_ready) {
    buf.S.alloc(static_cast<size_t>(cp) * ldg);
    CK(launch_gen_sketch_operator(buf.S.p, cp, ldg, c, m, seed, kind, sparse_nnz, st, stream_tag));
    launches += 1;
  }
  const int64_t wse = sketch_workspace_elems(m, n, cp);
  if (buf.ws.count < static_cast<size_t>(wse)) buf.ws.alloc(wse);
  CK(run_sketch_apply(A, m, n, lda, buf.S.p, ldg, cp, scale, Y, buf.ws.p, wse, stats, st, info));
  return launches + 4;
}

struct Workspace {
  DevBuf<double> Y, Wc, Wr, Bg, Ut, Yg, YgT, lu, part, sk_ws, S;
  DevBuf<uint8_t> col_mask, row_mask;
  DevBuf<char> state, lupp_scratch, qrcp_scratch;
  DevBuf<double> Wq;  // Y copy for the QRCP column selection (qrcp_pivot_cols takes W by value)
  DevBuf<int> commit_counter;  // arrivals of the U block's CTAs (fused commit), reset by the last
  DevBuf<double> At;  // row-major copy of A (n x m column-major, ld ldAt) for the row gathers A(I_k, :)
  int64_t ldAt = 0;
  DevBuf<double> scal;  // [0] asq, [1] ysq
  DevBuf<unsigned long long> nonfinite;
  char* h_state = nullptr;  // pinned mirror (thread-local cache, see pinned_state)
};

char* pinned_state(size_t bytes) {
  thread_local char* buf = nullptr;
  thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    CK(cudaMallocHost(reinterpret_cast<void**>(&buf), bytes));
    cap = bytes;
  }
  return buf;
}

void grow_factors(itercur_run* run, int64_t need, cudaStream_t st) {
  if (need <= run->capL) return;
  int64_t cap = std::max<int64_t>(run->capL * 2, need);
  const int64_t maxcap = std::min(run->m, run->sh.active ? run->sh.n_total : run->n) + run->bmax;
  cap = std::min(cap, maxcap);
  if (cap < need) cap = need;
  cap = (cap + 1) & ~int64_t(1);  // even: 16-byte aligned gathered columns (lean GEMM loads)
  DevBuf<double> L2, R2, D2;
  static const bool trace = env_flag("ITERCUR_HOST_TRACE");
  const auto t0 = std::chrono::steady_clock::now();
  L2.alloc(static_cast<size_t>(run->ldL) * cap);
  const auto t1 = std::chrono::steady_clock::now();
  R2.alloc(static_cast<size_t>(run->ldR) * cap);
  const auto t2 = std::chrono::steady_clock::now();
  D2.alloc(static_cast<size_t>(run->bmax) * cap);
  if (trace)
    fprintf(stderr, "[itercur grow] L %.0f MB in %.0fus, R~ %.0f MB in %.0fus, D in %.0fus\n",
            8e-6 * run->ldL * cap, std::chrono::duration<double, std::micro>(t1 - t0).count(), 8e-6 * run->ldR * cap,
            std::chrono::duration<double, std::micro>(t2 - t1).count(),
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t2).count());
  if (run->r > 0) {
    CK(cudaMemcpyAsync(L2.p, run->L.p, sizeof(double) * run->ldL * run->r, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(R2.p, run->Rt.p, sizeof(double) * run->ldR * run->r, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(D2.p, run->Dinv.p, sizeof(double) * run->bmax * run->r, cudaMemcpyDeviceToDevice, st));
  }
  // the copies and the old buffers' frees are ordered on st; waiting here only keeps the host from
  // running ahead of a regrowth (an empty run has nothing in flight to wait for)
  if (run->r > 0) CK(cudaStreamSynchronize(st));
  run->L.swap(L2);
  run->Rt.swap(R2);
  run->Dinv.swap(D2);
  run->capL = cap;
}

double min_margin(const double* best, const double* second, int count) {
  double mm = std::numeric_limits<double>::infinity();
  for (int s = 0; s < count; ++s)
    if (second[s] >= 0.0 && best[s] > 0.0) mm = std::min(mm, (best[s] - second[s]) / best[s]);
  return mm;
}

// The driver: proj/src/driver.cpp:48-167 over device state.
void run_iterative_cur(itercur_run* run) {
  const itercur_config& cfg = run->cfg;
  cudaStream_t st = run->wstream;
  const int64_t m = run->m, n = run->n, lda = run->lda;  // n: the columns this process holds
  const double* A = run->A;
  const auto t_start = std::chrono::steady_clock::now();
  // column sharding; an unsharded run is one local shard covering A
  ShardSpec& sh = run->sh;
  if (!sh.active) {
    sh.nloc = 1;
    sh.goff.assign(1, 0);
    sh.cnt.assign(1, n);
    sh.n_total = n;
  }
  const int64_t n_glob = sh.n_total;
  const bool emul = sh.emulated(), use_nccl = sh.active && sh.comm != nullptr;
  const NcclApi* nc = use_nccl ? nccl_api() : nullptr;
  if (use_nccl && !nc) fail(ITERCUR_E_CUDA, std::string("NCCL unavailable: ") + nccl_load_error());
  auto nck = [&](ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(ITERCUR_E_CUDA, std::string("NCCL error '") + nc->GetErrorString(r) + "' (" + what + ")");
  };
  // a local shard's first column within this process's A / Y / R~ (emulation: all columns are local)
  auto loc = [&](int s) -> int64_t { return emul ? sh.goff[s] : 0; };
  // sum of host scalars over the ranks (NCCL mode; a no-op otherwise)
  DevBuf<double> red;
  red.alloc(4);
  auto allreduce_host = [&](double* v, int k) {
    if (!use_nccl) return;
    CK(cudaMemcpyAsync(red.p, v, sizeof(double) * k, cudaMemcpyHostToDevice, st));
    nck(nc->AllReduce(red.p, red.p, k, ncclDouble, ncclSum, sh.comm, st), "allreduce scalars");
    CK(cudaMemcpyAsync(v, red.p, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  };
  auto count_nonfinite_all = [&]() -> double {
    DevBuf<unsigned long long> cnt;
    cnt.alloc(1);
    CK(launch_count_nonfinite(A, m, n, lda, cnt.p, st));
    run->launches += 1;
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double hv = static_cast<double>(h);
    allreduce_host(&hv, 1);
    return hv;
  };

  // ---- validation (driver.cpp:51-54, sketch.cpp:11-13), in the reference's order ----
  if (m == 0 || n == 0) fail(ITERCUR_E_INVALID_ARGUMENT, "matrix must be nonempty");
  if (m < 0 || n < 0 || lda < std::max<int64_t>(m, 1)) fail(ITERCUR_E_INVALID_ARGUMENT, "invalid matrix shape");
  const bool cheap_fail = cfg.epsilon < 0.0 || cfg.b < 1 || cfg.b > m;
  if (cheap_fail) {
    double asq = device_sumsq(A, m, n, lda, st);
    allreduce_host(&asq, 1);
    if (!std::isfinite(asq)) {
      if (count_nonfinite_all() > 0) fail(ITERCUR_E_INVALID_ARGUMENT, "matrix contains non-finite entries");
    }
    if (asq == 0.0) fail(ITERCUR_E_INVALID_ARGUMENT, "matrix must be nonzero");
    if (cfg.epsilon < 0.0) fail(ITERCUR_E_INVALID_ARGUMENT, "epsilon must be nonnegative");
    if (cfg.b < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "block size must be at least 1");
    fail(ITERCUR_E_INVALID_ARGUMENT, "block exceeds row count");
  }

  const int64_t b = cfg.b;
  const int64_t min_dim = std::min(m, n_glob);
  const int64_t max_rank = cfg.max_rank > 0 ? std::min(cfg.max_rank, min_dim) : min_dim;
  const int64_t max_iters = cfg.max_iters > 0 ? cfg.max_iters : (min_dim + b - 1) / b + 1;
  const int64_t c = cfg.sketch_rows > 0 ? cfg.sketch_rows : sketch_rows(b);
  if (c < b) fail(ITERCUR_E_INVALID_ARGUMENT, "sketch rows must be at least the block size");
  const int64_t cp = round_up(c, 8);
  run->c = c;
  run->cp = cp;
  run->bmax = b;
  run->ldL = even(m);
  run->ldR = even(n);

  Events evs;
  evs.on = cfg.profile != 0;
  Workspace ws;
  const int nloc = sh.nloc;
  const int B = static_cast<int>(b);
  const int kBatch = cfg.observer ? 1 : 8;  // iterations per batch graph (see the loop control below)
  const int64_t ldn = even(n), ldm = even(m);
  // ITERCUR_HOST_TRACE: where the host's set-up time goes
  static const bool setup_trace = env_flag("ITERCUR_HOST_TRACE");
  auto t_mark = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!setup_trace) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[itercur setup] %s %.0fus\n", what,
            std::chrono::duration<double, std::micro>(now - t_mark).count());
    t_mark = now;
  };
  // The run's large buffers first (factor capacity, the row-major copy of A), then the small
  // workspaces: the pool then serves the GB-sized requests from the previous runs' freed blocks of
  // the same sizes before small requests have carved them up.
  run->capL = 0;
  {
    // factor capacity: the whole max_rank + b up front when it is a small share of free HBM
    // (no regrowth copies, one graph capture per run), else grow by doubling
    const int64_t full = max_rank + b;
    const double full_bytes = 8.0 * static_cast<double>(run->ldL + run->ldR + b) * static_cast<double>(full);
    // free memory is only queried when the answer can depend on it: a capacity above a quarter of
    // the device's TOTAL memory (configs 3/4 without a rank cap) grows by doubling whatever is free.
    // cudaMemGetInfo sits on the run's critical path (~0.1 ms, at times milliseconds beside NVML
    // readers or large frees).
    static std::atomic<size_t> total_mem[kMaxDevices] = {};
    const int dev_ix = current_device();
    size_t free_b = 0, total_b = total_mem[dev_ix].load();
    bool have_free = false;
    if (total_b == 0) {
      CK(cudaMemGetInfo(&free_b, &total_b));
      total_mem[dev_ix].store(total_b);
      have_free = true;
    }
    bool fits = full_bytes <= 0.25 * static_cast<double>(total_b);
    if (fits) {
      if (!have_free) CK(cudaMemGetInfo(&free_b, &total_b));
      fits = full_bytes <= 0.25 * static_cast<double>(free_b);
      mark("cudaMemGetInfo");
    }
    int64_t first = fits ? full : std::min<int64_t>(full, std::max<int64_t>(kBatch * b, 256));
    if (use_nccl) {
      // the capacity sizes the packed block every rank allreduces (and the graphs' shapes): the
      // ranks' free memory differs with their shards, so they agree on the smallest choice
      double v = static_cast<double>(first);
      CK(cudaMemcpyAsync(red.p, &v, sizeof(double), cudaMemcpyHostToDevice, st));
      nck(nc->AllReduce(red.p, red.p, 1, ncclDouble, ncclMin, sh.comm, st), "allreduce capacity");
      CK(cudaMemcpyAsync(&v, red.p, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      first = static_cast<int64_t>(v);
    }
    grow_factors(run, first, st);
  }
  // row-major copy of A (when it is a modest share of free HBM): the U block's base A(I_k, :)
  // then reads |I_k| contiguous rows instead of one DRAM burst per element (~8 us per
  // iteration at config 2).
  // Made up front for A <= 2 GB (transpose <= ~0.6 ms; config 2: 32.3 ms eager vs 33.1 lazy after
  // 24 iterations — the lazy path's 1.6 GB pool allocation stalls the host between batches);
  // larger matrices skip it unless forced (config 3, 8 iterations, would pay 6 ms for 20 GB).
  // ITERCUR_ROWMAJOR_A=1 forces it, ITERCUR_NO_ROWMAJOR_A=1 disables it.
  static const bool at_off = env_flag("ITERCUR_NO_ROWMAJOR_A"), at_force = env_flag("ITERCUR_ROWMAJOR_A");
  auto maybe_make_rowmajor_a = [&](int64_t iters_done) -> bool {
    if (at_off || ws.At.p || iters_done > 0) return false;
    const double bytes = 8.0 * static_cast<double>(ldn) * static_cast<double>(m);
    if (!at_force && bytes > 2e9) return false;
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    if (bytes > 0.3 * static_cast<double>(free_b)) return false;
    mark("before the row-major copy's allocation");
    ws.At.alloc(static_cast<size_t>(ldn) * m);
    mark("row-major copy allocated");
    ws.ldAt = ldn;
    CK(launch_transpose(A, m, n, lda, ws.At.p, ldn, st));
    run->launches += 1;
    return true;
  };
  const bool at_early = maybe_make_rowmajor_a(0);
  (void)at_early;
  mark("factor capacity and row-major copy");
  ws.scal.alloc(2 * nloc + 2);
  ws.Y.alloc(static_cast<size_t>(cp) * n);

  // ---- sketch (make_sketch, sketch.cpp:10-24), ||A|| fused; one apply per local shard (the
  //      operator is regenerated from (seed, i) wherever it is needed) ----
  cudaEvent_t e_sk0 = evs.get(0), e_sk1 = evs.get(1);
  // enqueued once every buffer of the run is allocated, so the pool's requests are made on an idle
  // stream as they always were (allocating while the sketch ran would hide ~0.2 ms more, but was
  // only measured on boxes whose GB-sized pool requests took milliseconds either way)
  auto enqueue_sketch = [&]() {
    CK(cudaEventRecord(e_sk0, st));
    {
      const int kind = cfg.sketch_kind == ITERCUR_SKETCH_SPARSE_SIGN ? kSketchSparseSign : kSketchGaussian;
      SketchBuffers sb;
      for (int sI = 0; sI < nloc; ++sI) {
        SketchStats stats{ws.scal.p + 2 * sI, ws.scal.p + 2 * sI + 1};
        run->launches += apply_sketch(A + loc(sI) * lda, m, sh.cnt[sI], lda, kind, cfg.sparse_nnz, cfg.seed,
                                      cfg.sketch_stream > 0 ? static_cast<uint32_t>(cfg.sketch_stream) : kStreamSketch,
                                      c, cp, ws.Y.p + loc(sI) * cp, stats, sb, st, nullptr, sI > 0 && sb.S.p != nullptr);
      }
    }
    CK(cudaEventRecord(e_sk1, st));
    ws.S.reset();
    ws.sk_ws.reset();
  };
  // per-method floors (SelectionMethod::pivot_floor, select.hpp:12-15)
  const double col_floor = cfg.pivot_floor;
  const double row_floor = cfg.row_pivot_floor > 0.0 ? cfg.row_pivot_floor : cfg.pivot_floor;
  // The host's read of the sketch's norms — the zero / non-finite checks, rho_0 and the loop
  // control's initial state — is deferred until the workspaces are set up and the first batch's
  // graph is captured, instantiated and uploaded: all of that is independent of the data and
  // runs on the host while the device streams A through the sketch (config 4: ~0.7 ms of device
  // idle time between the sketch and the first iteration otherwise). The checks keep the
  // reference's order (driver.cpp:51-54, then the first select_* call's validation).
  double hs[2] = {0, 0};
  double ga_norm = 0.0, threshold = 0.0, rho = 1.0;
  std::function<void()> upload_ctl;  // set once the loop control's buffers exist
  auto finish_sketch = [&]() -> bool {
    {
      std::vector<double> hp(2 * nloc);
      CK(cudaMemcpyAsync(hp.data(), ws.scal.p, sizeof(double) * 2 * nloc, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int sI = 0; sI < nloc; ++sI) {  // shard order (fixed)
        hs[0] += hp[2 * sI];
        hs[1] += hp[2 * sI + 1];
      }
      allreduce_host(hs, 2);
    }
    if (!std::isfinite(hs[0])) {
      if (count_nonfinite_all() > 0) fail(ITERCUR_E_INVALID_ARGUMENT, "matrix contains non-finite entries");
    }
    if (hs[0] == 0.0) fail(ITERCUR_E_INVALID_ARGUMENT, "matrix must be nonzero");
    run->a_norm = std::sqrt(hs[0]);
    ga_norm = std::sqrt(hs[1]);
    run->ga_norm = ga_norm;
    run->sketch_s = elapsed_s(e_sk0, e_sk1);

    threshold = cfg.risk_adjust ? adjusted_threshold_impl(cfg.epsilon, cfg.delta, cfg.alpha, c) : cfg.epsilon;
    run->threshold = threshold;

    // rho_0 (downdate with empty factors, sketch.cpp:27-30)
    rho = ga_norm > 0.0 ? 1.0 : 0.0;
    if (rho <= threshold) {
      run->status = ITERCUR_CONVERGED;
      run->final_rho = rho;
      run->note = "threshold at or above the initial estimate; empty factorization";
      // nothing was selected: the factor buffers set up ahead of this check go back to the pool
      run->L.reset();
      run->Rt.reset();
      run->Dinv.reset();
      run->capL = 0;
      run->total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      return false;
    }
    // the reference validates the selection methods on the first select_* call; the column
    // method is validated first, as select_columns runs before select_rows (select.cpp:24-28)
    if (!(col_floor > 0.0 && col_floor < 1.0)) fail(ITERCUR_E_INVALID_ARGUMENT, "pivot_floor must lie in (0, 1)");
    if (!(row_floor > 0.0 && row_floor < 1.0)) fail(ITERCUR_E_INVALID_ARGUMENT, "pivot_floor must lie in (0, 1)");
    check_method(cfg.col_method);
    check_method(cfg.row_method);
    upload_ctl();
    return true;
  };

  // ---- workspaces ----
  // ldn: this process's columns (Y, R~, the U block); ldng: the replicated Wc over all columns
  // (NCCL mode: room for world equal blocks, so Wc's rows gather in place column by column)
  const int64_t blk = use_nccl ? shard_block(n_glob, sh.world) : 0;  // rank r owns [r*blk, min((r+1)*blk, n))
  const int64_t ldng = use_nccl ? std::max(even(n_glob), blk * sh.world) : even(n_glob);
  ws.Wc.alloc(static_cast<size_t>(ldng) * B);
  ws.Wr.alloc(static_cast<size_t>(ldm) * B);
  ws.Ut.alloc(static_cast<size_t>(ldn) * B);
  ws.Yg.alloc(static_cast<size_t>(B) * cp);
  ws.YgT.alloc(static_cast<size_t>(even(B)) * cp);  // Y(:, J_k)^T for the unfused downdate (k-contiguous)
  ws.col_mask.alloc(n_glob);
  ws.row_mask.alloc(m);
  CK(cudaMemsetAsync(ws.col_mask.p, 0, n_glob, st));
  CK(cudaMemsetAsync(ws.row_mask.p, 0, m, st));
  ws.lupp_scratch.alloc(lupp_scratch_bytes(B));
  CK(lupp_scratch_init(ws.lupp_scratch.p, st));
  const bool col_qrcp = cfg.col_method == ITERCUR_PIVOT_QRCP, row_qrcp = cfg.row_method == ITERCUR_PIVOT_QRCP;
  if (sh.active && (col_qrcp || row_qrcp))
    fail(ITERCUR_E_INVALID_ARGUMENT, "column-sharded runs support LUPP selection only");
  if (col_qrcp || row_qrcp) ws.qrcp_scratch.alloc(qrcp_scratch_bytes());
  if (col_qrcp) ws.Wq.alloc(static_cast<size_t>(cp) * n);
  // iterations are enqueued in batches of kBatch without a host round trip; the loop control
  // (budgets, stop tests, rank) lives on the device (IterCtl), and every kernel of an
  // iteration after the stop returns immediately.
  // With an IterationObserver every batch is one iteration, so the observer sees each
  // iteration's factors (driver.cpp:154) before the next one starts.
  const size_t slot_bytes = round_up(iter_state_bytes(B), 64);
  ws.state.alloc(slot_bytes * kBatch + sizeof(IterCtl));
  char* slots = ws.state.p;
  IterCtl* d_ctl = reinterpret_cast<IterCtl*>(ws.state.p + slot_bytes * kBatch);
  ws.h_state = pinned_state(slot_bytes * kBatch + sizeof(IterCtl));
  upload_ctl = [&, d_ctl, slot_bytes, kBatch, B]() {  // from finish_sketch, once the norms are on the host
    IterCtl h{};
    h.r = 0;
    h.k = 0;
    h.max_rank = max_rank;
    h.max_iters = max_iters;
    h.done = 0;
    h.status = ITERCUR_MAX_RANK;
    h.b = B;
    h.ysq = hs[1];
    h.rho = rho;
    h.threshold = threshold;
    h.ga_norm = ga_norm;
    IterCtl* hc = reinterpret_cast<IterCtl*>(ws.h_state + slot_bytes * kBatch);
    *hc = h;
    CK(cudaMemcpyAsync(d_ctl, hc, sizeof(IterCtl), cudaMemcpyHostToDevice, st));
  };
  // QRCP rows are not in pivot order: D_k is factored with partial pivoting (cross_lu) and
  // its permutation kept per block for the solves and the core export
  if (row_qrcp) run->Piv.alloc(std::max<int64_t>(max_rank + b, 1));
  run->dI.alloc(std::max<int64_t>(max_rank + b, 1));
  run->dJ.alloc(std::max<int64_t>(max_rank + b, 1));
  ws.Bg.alloc(static_cast<size_t>(run->capL) * B);
  // sharded runs: the selected block's columns [A(:,J_k) | R~(0:r,J_k) | Y(:,J_k)] assembled from
  // their owners (NCCL: one sum-allreduce of disjoint contributions; emulation: each shard writes
  // its own columns), replacing the single-device gathers
  DevBuf<double> pack;
  int64_t pack_ldr = 0;
  auto alloc_pack = [&]() {
    if (!sh.active) return;
    pack_ldr = run->capL;
    pack.alloc(static_cast<size_t>(ldm + pack_ldr + cp) * B);
  };
  alloc_pack();
  auto packA = [&]() { return pack.p; };
  auto packR = [&]() { return pack.p + ldm * B; };
  auto packY = [&]() { return pack.p + (ldm + pack_ldr) * B; };
  // optional U-block trace (ITERCUR_UB_TRACE=k: phases and CTA spans at iteration k)
  const char* ub_trace_env = getenv("ITERCUR_UB_TRACE");
  const int64_t ub_trace_k = ub_trace_env ? atoll(ub_trace_env) : 0;
  DevBuf<long long> ub_dbg;
  if (ub_trace_env) {
    ub_dbg.alloc(32 + 2 * 8192);
    CK(cudaMemsetAsync(ub_dbg.p, 0, sizeof(long long) * (32 + 2 * 8192), st));
  }
  // the same trace for the row-residual GEMM (ITERCUR_G1_TRACE=k)
  const char* g1_trace_env = getenv("ITERCUR_G1_TRACE");
  const int64_t g1_trace_k = g1_trace_env ? atoll(g1_trace_env) : 0;
  DevBuf<long long> g1_dbg;
  if (g1_trace_env) {
    g1_dbg.alloc(32 + 2 * 8192);
    CK(cudaMemsetAsync(g1_dbg.p, 0, sizeof(long long) * (32 + 2 * 8192), st));
  }
  // the row-residual GEMM: S_row = A(:,J_k) - L * Rt(:,J_k) into L's next columns and the row LUPP input
  auto gemm1_params = [&](int64_t ldbg, IterState* slot, const IterArrays& arr) {
    TsGemmParams p;
    p.M = m;
    p.K = ldbg;
    p.ctl = d_ctl;
    p.k_from_r = 1;
    p.N = B;
    p.d_n = &slot->ncols;
    p.A = run->L.p;
    p.lda = run->ldL;
    p.B = ws.Bg.p;  // B(k, q) = Rt(k, J_k[q])
    p.bsk = 1;
    p.bsn = ldbg;
    p.base_mode = kBaseGatherCols;
    p.src = A;
    p.lds = lda;
    p.idx = arr.col_idx;
    if (sh.active) {  // the assembled block: base A(:, J_k) and R~(:, J_k) contiguous
      p.B = packR();
      p.base_mode = kBaseContigCols;
      p.src = packA();
      p.lds = ldm;
      p.col0 = 0;
      p.idx = nullptr;
    }
    p.alpha = -1.0;
    p.out_mode = kOutColMajor;
    p.C0 = run->L.p;
    p.c0_off_per_r = run->ldL;
    p.ldc0 = run->ldL;
    p.C1 = ws.Wr.p;
    p.ldc1 = ldm;
    p.dbg = g1_dbg.p;
    p.dbg_k = g1_trace_k;
    return p;
  };
  // the fused U-block kernel (GEMM2 + solves + downdate) when the shape qualifies
  // per local shard: its columns of Y / R~ / A (this process's buffers at column loc(s)) and its
  // rows of the replicated Wc (global offset goff[s]); the ||Y||^2 partials of shard s at poff[s]
  std::vector<int64_t> poff(nloc + 1, 0);
  auto ublock_params = [&](int64_t ldbg, IterState* slot, const IterArrays& arr, int sI) {
    const int64_t lo = loc(sI);
    TsGemmParams p;
    p.M = sh.cnt[sI];
    p.K = ldbg;
    p.ctl = d_ctl;
    p.k_from_r = 1;
    p.N = B;
    p.d_n = &slot->width;
    p.A = run->Rt.p + lo;
    p.lda = run->ldR;
    p.B = ws.Bg.p;  // B(k, q) = L(I_k[q], k)
    p.bsk = 1;
    p.bsn = ldbg;
    if (ws.At.p) {  // A(I_k[q], j) = At(j, I_k[q])
      p.base_mode = kBaseGatherCols;
      p.src = ws.At.p + lo;
      p.lds = ws.ldAt;
    } else {
      p.base_mode = kBaseGatherRowsT;
      p.src = A + lo * lda;
      p.lds = lda;
    }
    p.idx = arr.row_idx;
    p.alpha = -1.0;
    p.out_mode = kOutNone;
    p.lu = run->Dinv.p;
    p.ldd = run->bmax;
    p.rt = run->Rt.p + lo;
    p.ldr = run->ldR;
    p.yg = sh.active ? packY() : ws.Yg.p;
    p.ycp = static_cast<int>(cp);
    p.y = ws.Y.p + lo * cp;
    p.Wc = ws.Wc.p + sh.goff[sI];
    p.ldwc = ldng;
    p.wc_rows = B;
    p.norm_part = ws.part.p + poff[sI];
    p.dbg = ub_dbg.p;
    p.dbg_k = ub_trace_k;
    return p;
  };
  const bool fused_ub = !env_flag("ITERCUR_NO_FUSED_UBLOCK") && !row_qrcp && [&] {
    IterState* slot0 = reinterpret_cast<IterState*>(slots);
    bool ok = (run->capL & 1) == 0;
    for (int sI = 0; sI < nloc && ok; ++sI) {
      TsGemmParams p = ublock_params(run->capL, slot0, iter_arrays(slot0, B), sI);
      p.norm_part = reinterpret_cast<double*>(16);  // placeholder: allocated below
      ok = ts_gemm_ublock_supported(p);
    }
    return ok;
  }();
  for (int sI = 0; sI < nloc; ++sI)
    poff[sI + 1] = poff[sI] + (fused_ub ? ts_gemm_ublock_parts(sh.cnt[sI]) : ts_gemm_grid_size(sh.cnt[sI], static_cast<int>(cp)));
  const int64_t y_parts = poff[nloc];
  ws.part.alloc(std::max<int64_t>(y_parts, 1) + 1);  // + the rank-local sum (NCCL mode)
  ws.commit_counter.alloc(1);
  CK(cudaMemsetAsync(ws.commit_counter.p, 0, sizeof(int), st));
  // NCCL mode: the ranks' rows of Wc gathered in place, one allgather per column (equal blocks)
  auto allgather_wc = [&]() {
    if (!use_nccl) return;
    nck(nc->GroupStart(), "group start");
    for (int h = 0; h < B; ++h)
      nck(nc->AllGather(ws.Wc.p + h * ldng + sh.rank * blk, ws.Wc.p + h * ldng, blk, ncclDouble, sh.comm, st),
          "allgather Wc");
    nck(nc->GroupEnd(), "group end");
  };

  mark("workspaces");
  enqueue_sketch();
  mark("sketch enqueued");
  // initial Wc = Y^T(:, 0:b)
  for (int sI = 0; sI < nloc; ++sI) {
    CK(launch_transpose_rows(ws.Y.p + loc(sI) * cp, cp, sh.cnt[sI], B, ws.Wc.p + sh.goff[sI], ldng, st));
    run->launches += 1;
  }
  allgather_wc();

  const uint8_t epoch = 2;  // the global-memory LUPP clears its in-call marks, so one epoch suffices
  static uint32_t run_counter = 0;
  const uint32_t gen_base = ((++run_counter) & 0x3FFu) << 21;  // LUPP slot-tag generations
  const bool use_graph = !evs.on && !env_flag("ITERCUR_NO_GRAPH");
  // batch graphs by split plan (they differ only in the GEMMs' K-split counts), valid for one
  // factor capacity and one U-block base; the next batch's graph is captured while the current
  // one runs on the device
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
  };
  struct GraphCache {
    std::vector<std::pair<int64_t, GraphEntry>> v;
    GraphEntry* find(int64_t sig) {
      for (auto& e : v)
        if (e.first == sig) return &e.second;
      return nullptr;
    }
    void clear() {
      for (auto& e : v) cudaGraphExecDestroy(e.second.exec);
      v.clear();
    }
    ~GraphCache() { clear(); }
  } graphs;
  int64_t graph_cap = -1;
  int64_t k_host = 0, r_host = 0, observed = 0;
  int64_t ev_i = 2;
  std::vector<size_t> iter_events;
  bool done = false;
  static const bool host_trace = env_flag("ITERCUR_HOST_TRACE");
  bool sketch_pending = true;
  const double setup_us =
      std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_start).count();
  using hclock = std::chrono::steady_clock;
  auto us_since = [](hclock::time_point t0) {
    return std::chrono::duration<double, std::micro>(hclock::now() - t0).count();
  };
  while (!done) {
    const auto tb0 = hclock::now();
    double t_grow = 0, t_capture = 0, t_launch = 0, t_sync = 0;
    // capacity for a whole batch
    const int64_t need = std::min(r_host + static_cast<int64_t>(kBatch) * b, max_rank + b);
    if (need > run->capL) {
      grow_factors(run, need, st);
      ws.Bg.alloc(static_cast<size_t>(run->capL) * B);
      alloc_pack();
      t_grow = us_since(tb0);
    }
    const bool at_new = maybe_make_rowmajor_a(k_host);  // (re-capture: the U block's base changes)
    const int64_t ldbg = run->capL;
    // the GEMMs' K-split counts are planned for the largest K this batch can reach (the kernels
    // take K from the device loop control): few splits while the factors are thin. The batch
    // graph is re-captured only when a planned count changes.
    auto k_plan_for = [&](int64_t r0) {
      return std::max<int64_t>(1, std::min<int64_t>(ldbg, r0 + static_cast<int64_t>(kBatch) * b));
    };
    auto plan_sig_for = [&](int64_t kp) {
      IterState* slot0 = reinterpret_cast<IterState*>(slots);
      const IterArrays arr0 = iter_arrays(slot0, B);
      TsGemmParams g1 = gemm1_params(ldbg, slot0, arr0);
      g1.k_plan = kp;
      int64_t sig = ts_gemm_planned_splits(g1, false);
      if (fused_ub) {
        for (int sI = 0; sI < nloc; ++sI) {  // every shard's U block (their M may differ)
          TsGemmParams ub = ublock_params(ldbg, slot0, arr0, sI);
          ub.k_plan = kp;
          sig = sig * 131 + ts_gemm_planned_splits(ub, true);
        }
      }
      return sig;
    };
    int64_t k_plan = k_plan_for(r_host);
    const int64_t plan_sig = plan_sig_for(k_plan);
    // the iteration kernels of one batch; captured once into a CUDA graph (re-captured only
    // when the factor buffers grow) and replayed, so a batch costs one graph launch
    int64_t batch_launches = 0;
    // iteration-begin + gathers folded into the cluster LUPP kernels: measured slightly slower
    // than separate grid-wide gather launches inside the batch graphs (config 2: 39.4 vs
    // 38.8 ms; the strided gathers then run on the cluster's 16 SMs only), so opt-in
    static const bool fuse_off = !env_flag("ITERCUR_LUPP_FUSION");
    // the iteration commit (||Y||^2 from the partials, stop tests, index append); NCCL mode: the
    // rank's partials summed in a fixed order, then summed over the ranks, then the commit; and the
    // ranks' rows of the downdated Wc gathered for the next column selection
    auto commit_iteration = [&](IterState* slot, const IterArrays& arr) {
      if (use_nccl) {
        double* mine = ws.part.p + y_parts;
        CK(launch_sum_partials(ws.part.p, y_parts, mine, st, d_ctl));
        nck(nc->AllReduce(mine, mine, 1, ncclDouble, ncclSum, sh.comm, st), "allreduce ||Y||^2");
        CK(launch_commit(d_ctl, slot, arr, run->dI.p, run->dJ.p, ws.row_mask.p, ws.col_mask.p, mine, 1, st));
        allgather_wc();
        batch_launches += 1;
      } else {
        CK(launch_commit(d_ctl, slot, arr, run->dI.p, run->dJ.p, ws.row_mask.p, ws.col_mask.p, ws.part.p, y_parts,
                         st));
      }
    };
    auto enqueue_batch = [&]() {
      // programmatic dependent launch along the iteration's kernel chain: measured neutral to
      // slightly slower inside the batch graphs on B200 (config 2: 38.5 vs 38.3 ms), so opt-in
      static const bool pdl = env_flag("ITERCUR_PDL");
      PdlScope pdl_scope(pdl && !evs.on);
      batch_launches = 0;
      for (int j = 0; j < kBatch; ++j) {
        IterState* slot = reinterpret_cast<IterState*>(slots + slot_bytes * j);
        const IterArrays arr = iter_arrays(slot, B);
        const size_t e0 = static_cast<size_t>(ev_i);
        if (evs.on) {
          CK(cudaEventRecord(evs.get(e0), st));
          iter_events.push_back(e0);
          ev_i += 6;
        }
        // (1) column selection: LUPP on W = Y^T (select_columns, select.cpp:121-139); on the
        //     cluster path the same kernel also opens the iteration (iter_begin) and, after its
        //     last pivot, gathers R~(:,J_k) (GEMM1's B) and Y(:,J_k) (the downdate's B)
        bool col_fused = false, begin_fused = false;
        {
          LuppArgs la{};
          la.W = ws.Wc.p;
          la.rows = n_glob;
          la.ldw = ldng;
          la.cols_max = B;
          la.d_steps = &d_ctl->block;
          la.mask = ws.col_mask.p;
          la.epoch = epoch;
          la.d_norm_sq = &d_ctl->ysq;
          la.pivot_floor = col_floor;
          la.d_idx = arr.col_idx;
          la.d_best = arr.col_best;
          la.d_second = arr.col_second;
          la.d_count = &slot->ncols;
          la.d_gen_k = &d_ctl->k;
          la.gen_base = gen_base;
          la.gen_which = 0;
          const bool fusable = !col_qrcp && fused_ub && lupp_fuses_iteration_work(la);
          col_fused = fusable && !fuse_off && !sh.active;  // sharded: the block is packed instead
          // the iteration begin alone (no gathers) folded into the cluster LUPP
          // (measured: column-selection phase 6.90 -> 6.57 ms at config 2; ITERCUR_NO_LUPP_FUSE_BEGIN)
          static const bool begin_only = !env_flag("ITERCUR_NO_LUPP_FUSE_BEGIN");
          if (col_fused || (fusable && begin_only)) {
            la.begin_ctl = d_ctl;
            la.begin_slot = slot;
            begin_fused = true;
          } else {
            CK(launch_iter_begin(d_ctl, slot, st));
          }
          if (col_fused) {
            la.post[0] = {run->Rt.p, run->ldR, 1, ldbg, &d_ctl->r, ws.Bg.p, ldbg, B};
            la.post[1] = {ws.Y.p, 1, cp, cp, nullptr, ws.Yg.p, cp, B};
          }
          if (col_qrcp) {  // QRCP over the c-row columns of (a copy of) Y, select.cpp:79-117,121-139
            CK(cudaMemcpyAsync(ws.Wq.p, ws.Y.p, sizeof(double) * cp * n, cudaMemcpyDeviceToDevice, st));
            CK(run_qrcp(ws.Wq.p, n, static_cast<int>(c), nullptr, 1, cp, &d_ctl->block, B, ws.col_mask.p, epoch,
                        &d_ctl->ysq, col_floor, arr.col_idx, arr.col_best, arr.col_second, &slot->ncols,
                        nullptr, nullptr, ws.qrcp_scratch.p, d_ctl, st));
          } else {
            CK(run_lupp_with_scratch(la, ws.lupp_scratch.p, st, nullptr));
          }
        }
        if (evs.on) CK(cudaEventRecord(evs.get(e0 + 1), st));

        // (2) row residual S_row = A(:,J_k) - L * Rt(:,J_k)  (row_residual, sketch.cpp:43-60);
        //     Rt(:,J_k) is gathered once into a contiguous K x w block (a strided gather inside
        //     the GEMM loader would re-fetch one 32-B sector per element in every CTA)
        if (sh.active) {
          // the block's columns from their owners: A(:,J_k), R~(0:r,J_k), Y(:,J_k) (all of J_k
          // is replicated after the column selection); NCCL: one sum-allreduce of the packs
          for (int sI = 0; sI < nloc; ++sI) {
            const int64_t lo = loc(sI);
            CK(launch_pack_owned(d_ctl, &slot->ncols, arr.col_idx, B, sh.goff[sI], sh.cnt[sI], A + lo * lda, lda, m,
                                 run->Rt.p + lo, run->ldR, ldbg, ws.Y.p + lo * cp, cp, packA(), ldm, packR(), pack_ldr,
                                 packY(), use_nccl, st));
            batch_launches += 1;
          }
          if (use_nccl)
            nck(nc->AllReduce(pack.p, pack.p, static_cast<size_t>(ldm + pack_ldr + cp) * B, ncclDouble, ncclSum,
                              sh.comm, st),
                "allreduce block");
        } else if (!col_fused) {
          CK(launch_gather(run->Rt.p, run->ldR, 1, ldbg, arr.col_idx, &slot->ncols, B, ws.Bg.p, ldbg, st, d_ctl, true));
        }
        // Y(:, J_k) for the U block's downdate on a side branch: it needs only J_k, so it can run
        // beside the row residual and the row selection (joined before the U block). Measured
        // slower inside the batch graphs (config 2: 35.6 vs 32.6 ms; the concurrent kernel delays
        // the cluster launches), so opt-in: ITERCUR_SIDE_GATHER
        static const bool y_branch = env_flag("ITERCUR_SIDE_GATHER");
        const bool y_side = fused_ub && !col_fused && y_branch && !sh.active;
        if (y_side) {
          SideStream& ss = side_stream();
          CK(cudaEventRecord(ss.fork, st));
          CK(cudaStreamWaitEvent(ss.s, ss.fork, 0));
          CK(launch_gather(ws.Y.p, 1, cp, cp, arr.col_idx, &slot->ncols, B, ws.Yg.p, cp, ss.s, d_ctl, false));
          CK(cudaEventRecord(ss.join, ss.s));
        }
        {
          TsGemmParams p = gemm1_params(ldbg, slot, arr);
          p.k_plan = k_plan;
          CK(run_ts_gemm(p, st));
        }
        if (evs.on) CK(cudaEventRecord(evs.get(e0 + 2), st));

        int row_lupp_path = 0;
        bool row_fused = false;
        // (3) row selection: LUPP on S_row (select_rows, select.cpp:141-165), b = |cols|
        {
          LuppArgs la{};
          la.W = ws.Wr.p;
          la.rows = m;
          la.ldw = ldm;
          la.cols_max = B;
          la.d_steps = &slot->ncols;
          la.mask = ws.row_mask.p;
          la.epoch = epoch;
          la.d_norm_sq = nullptr;  // ||S_row||_F over its |cols| columns, computed in-kernel
          la.pivot_floor = row_floor;
          la.d_idx = arr.row_idx;
          la.d_best = arr.row_best;
          la.d_second = arr.row_second;
          la.d_count = &slot->nrows;
          la.d_width_out = &slot->width;  // width = min(|cols|, |rows|), driver.cpp:123
          la.d_width_cap = &slot->ncols;
          la.d_gen_k = &d_ctl->k;
          la.gen_base = gen_base;
          la.gen_which = 1;
          la.lu_out = run->Dinv.p;
          la.lu_ld = run->bmax;
          la.d_lu_r = &d_ctl->r;
          row_fused = !row_qrcp && fused_ub && !fuse_off && lupp_fuses_iteration_work(la);
          if (row_fused) la.post[0] = {run->L.p, run->ldL, 1, ldbg, &d_ctl->r, ws.Bg.p, ldbg, B};  // L(I_k, :)
          if (row_qrcp) {  // QRCP over the rows of S_row (select.cpp:141-165); D_k by cross_lu below
            row_lupp_path = 0;
            CK(run_qrcp(ws.Wr.p, m, B, &slot->ncols, ldm, 1, &slot->ncols, B, ws.row_mask.p, epoch, nullptr,
                        row_floor, arr.row_idx, arr.row_best, arr.row_second, &slot->nrows, &slot->width,
                        &slot->ncols, ws.qrcp_scratch.p, d_ctl, st));
          } else {
            CK(run_lupp_with_scratch(la, ws.lupp_scratch.p, st, &row_lupp_path));
          }
        }
        if (evs.on) CK(cudaEventRecord(evs.get(e0 + 3), st));

        // (4) core step: LU of D_k = S_row(I_k, 0:w); U_k^T = A(I_k,:)^T - Rt^T L(I_k,:)^T;
        //     Rt_k = D_k^{-1} U_k by row-wise LU solves (rows r..r+w of Rt)
        static const bool force_cross_lu = env_flag("ITERCUR_FORCE_CROSS_LU");  // A/B check
        if (row_lupp_path >= 0 || force_cross_lu)  // the cluster / panel LUPP emitted D_k's factors itself
          CK(launch_cross_lu(run->L.p, run->ldL, arr.row_idx, &slot->width, B, run->Dinv.p, run->bmax, st, d_ctl,
                             run->Piv.p));
        static const bool pair_off = env_flag("ITERCUR_NO_PAIR_GATHER");  // A/B
        const bool y_here = fused_ub && !y_side && !col_fused && !sh.active;  // Y(:, J_k) gathered before the U block
        if (!row_fused && y_here && !pair_off)  // L(I_k, :)^T and Y(:, J_k) in one launch
          CK(launch_gather_pair(run->L.p, run->ldL, 1, ldbg, arr.row_idx, ws.Bg.p, ldbg, true, ws.Y.p, 1, cp, cp,
                                arr.col_idx, ws.Yg.p, cp, false, &slot->width, B, st, d_ctl));
        else if (!row_fused)
          CK(launch_gather(run->L.p, run->ldL, 1, ldbg, arr.row_idx, &slot->width, B, ws.Bg.p, ldbg, st, d_ctl, true));
        if (fused_ub) {
          // Y(:, J_k) before the downdate, then one kernel: U_k^T, the solves against D_k,
          // R~ rows, Y^T -= R~_k^T Y(:, J_k)^T, ||Y||^2 partials and Wc
          if (y_side)
            CK(cudaStreamWaitEvent(st, side_stream().join, 0));
          else if (y_here && (row_fused || pair_off))
            CK(launch_gather(ws.Y.p, 1, cp, cp, arr.col_idx, &slot->width, B, ws.Yg.p, cp, st, d_ctl, false));
          TsGemmParams p = ublock_params(ldbg, slot, arr, 0);
          p.k_plan = k_plan;
          // the commit in the U block's last CTA instead of its own kernel: measured slower
          // (config 2 phase sums 32.17 vs 31.60 ms: every CTA's release fence before its arrival
          // lengthens the kernel more than the launch it saves), so opt-in: ITERCUR_FUSED_COMMIT
          static const bool fused_commit_env = env_flag("ITERCUR_FUSED_COMMIT");
          const bool fused_commit = fused_commit_env && !sh.active;
          if (fused_commit) {
            p.commit.ctl = d_ctl;
            p.commit.slot = slot;
            p.commit.row_idx = arr.row_idx;
            p.commit.col_idx = arr.col_idx;
            p.commit.I_all = run->dI.p;
            p.commit.J_all = run->dJ.p;
            p.commit.row_mask = ws.row_mask.p;
            p.commit.col_mask = ws.col_mask.p;
            p.commit.counter = ws.commit_counter.p;
          }
          CK(run_ts_gemm_ublock(p, st));
          for (int sI = 1; sI < nloc; ++sI) {  // the other local shards' U blocks (emulation)
            TsGemmParams ps = ublock_params(ldbg, slot, arr, sI);
            ps.k_plan = k_plan;
            CK(run_ts_gemm_ublock(ps, st));
          }
          batch_launches += 9 + (row_lupp_path >= 0 ? 1 : 0) - (col_fused ? 2 : 0) - (begin_fused ? 1 : 0) -
                            (row_fused ? 1 : 0) - ((!row_fused && y_here && !pair_off) ? 1 : 0) + (nloc - 1) -
                            (sh.active ? 2 : 0);
          if (evs.on) CK(cudaEventRecord(evs.get(e0 + 4), st));
          if (evs.on) CK(cudaEventRecord(evs.get(e0 + 5), st));  // downdate fused into the core step
          if (!fused_commit) {
            commit_iteration(slot, arr);
          } else {
            batch_launches -= 1;
          }
          continue;
        }
        for (int sI = 0; sI < nloc; ++sI) {
          const int64_t lo = loc(sI);
          TsGemmParams p;
          p.M = sh.cnt[sI];
          p.K = ldbg;
          p.ctl = d_ctl;
          p.k_from_r = 1;
          p.N = B;
          p.d_n = &slot->width;
          p.A = run->Rt.p + lo;
          p.lda = run->ldR;
          p.B = ws.Bg.p;  // B(k, q) = L(I_k[q], k)
          p.bsk = 1;
          p.bsn = ldbg;
          if (ws.At.p) {
            p.base_mode = kBaseGatherCols;
            p.src = ws.At.p + lo;
            p.lds = ws.ldAt;
          } else {
            p.base_mode = kBaseGatherRowsT;
            p.src = A + lo * lda;
            p.lds = lda;
          }
          p.idx = arr.row_idx;
          p.alpha = -1.0;
          p.out_mode = kOutColMajor;
          p.C0 = ws.Ut.p + lo;
          p.ldc0 = ldn;
          CK(run_ts_gemm(p, st));
          CK(launch_rows_lu_solve(ws.Ut.p + lo, ldn, sh.cnt[sI], run->Dinv.p, run->bmax, &slot->width, B,
                                  run->Rt.p + lo, run->ldR, st, d_ctl, run->ldR, run->Piv.p));
        }
        if (evs.on) CK(cudaEventRecord(evs.get(e0 + 4), st));

        // (5) downdate Y -= Y(:,J_k) * Rt_k in place (downdate_col_residual, sketch.cpp:26-41),
        //     ||Y||^2 fused, Wc = Y^T(:, 0:b) for the next column selection
        // Y(:, J_k) gathered transposed (w x cp, k-contiguous): the downdate then runs the lean
        // cp.async loop instead of the generic loader (config 4: 118 -> ~60 us per iteration)
        const int64_t ldq = even(B);
        if (!sh.active) {
          CK(launch_gather(ws.Y.p, 1, cp, cp, arr.col_idx, &slot->width, B, ws.YgT.p, ldq, st, d_ctl, false, true));
        }
        for (int sI = 0; sI < nloc; ++sI) {
          const int64_t lo = loc(sI);
          TsGemmParams p;
          p.M = sh.cnt[sI];
          p.K = B;
          p.d_k = &slot->width;
          p.ctl = d_ctl;
          p.N = static_cast<int>(cp);
          p.A = run->Rt.p + lo;
          p.a_off_per_r = run->ldR;
          p.lda = run->ldR;
          if (sh.active) {
            p.B = packY();  // B(q, h) = Y(h, J[q]) = PackY[h + q * cp]
            p.bsk = cp;
            p.bsn = 1;
          } else {
            p.B = ws.YgT.p;  // B(q, h) = Y(h, J[q]) = YgT[q + h * ldq]
            p.bsk = 1;
            p.bsn = ldq;
          }
          p.base_mode = kBaseInPlaceRowMajor;
          p.alpha = -1.0;
          p.out_mode = kOutRowMajor;
          p.C0 = ws.Y.p + lo * cp;
          p.ldc0 = cp;
          p.Wc = ws.Wc.p + sh.goff[sI];
          p.ldwc = ldng;
          p.wc_rows = B;
          p.norm_part = ws.part.p + poff[sI];
          CK(run_ts_gemm(p, st));
        }
        commit_iteration(slot, arr);
        batch_launches += 11 + (row_lupp_path >= 0 ? 1 : 0) + 3 * (nloc - 1) - (sh.active ? 2 : 0);
        if (evs.on) CK(cudaEventRecord(evs.get(e0 + 5), st));
      }
    };
    const auto tc0 = hclock::now();
    auto capture = [&](int64_t kp) {
      k_plan = kp;
      GraphEntry e;
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_batch();
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CK(cudaStreamEndCapture(st, &g));
      const cudaError_t ie = cudaGraphInstantiate(&e.exec, g, 0);
      cudaGraphDestroy(g);
      CK(ie);
      e.launches = batch_launches;
      return e;
    };
    GraphEntry* ge = nullptr;
    if (use_graph) {
      if (graph_cap != run->capL || at_new) {
        graphs.clear();
        graph_cap = run->capL;
      }
      ge = graphs.find(plan_sig);
      if (!ge) {
        graphs.v.emplace_back(plan_sig, capture(k_plan));
        ge = &graphs.v.back().second;
        // first batch: the sketch is still running — place the executable graph on the device now
        // (on the side stream), so its launch after the norm checks costs microseconds
        if (sketch_pending) {
          SideStream& ss = side_stream();
          if (cudaGraphUpload(ge->exec, ss.s) == cudaSuccess) {
            CK(cudaEventRecord(ss.join, ss.s));
            CK(cudaStreamWaitEvent(st, ss.join, 0));
          } else {
            cudaGetLastError();
          }
        }
        t_capture = us_since(tc0);
      }
    }
    if (sketch_pending) {  // the norm checks, rho_0 and the loop control's upload (see finish_sketch)
      sketch_pending = false;
      const auto tf0 = hclock::now();
      if (!finish_sketch()) return;
      if (host_trace)
        fprintf(stderr, "[itercur setup] %.0fus before the first batch (sketch %.0fus, waited %.0fus for it)\n",
                us_since(tb0) + setup_us, run->sketch_s * 1e6, us_since(tf0));
    }
    const auto tl0 = hclock::now();
    if (use_graph) {
      CK(cudaGraphLaunch(ge->exec, st));
      batch_launches = ge->launches;
    } else {
      enqueue_batch();
    }
    t_launch = us_since(tl0);
    run->launches += batch_launches;
    // one D2H read per batch: the batch's records + the loop control
    CK(cudaMemcpyAsync(ws.h_state, ws.state.p, slot_bytes * kBatch + sizeof(IterCtl), cudaMemcpyDeviceToHost, st));
    // while the device runs this batch: the graph of the next batch's plan (its K bound is at
    // most r + 2 batches of b), if the capacity will not have to grow first
    if (use_graph && std::min(r_host + 2 * static_cast<int64_t>(kBatch) * b, max_rank + b) <= run->capL) {
      const int64_t kn = k_plan_for(r_host + static_cast<int64_t>(kBatch) * b);
      const int64_t sn = plan_sig_for(kn);
      if (!graphs.find(sn)) {
        const auto tp = hclock::now();
        graphs.v.emplace_back(sn, capture(kn));
        t_capture += us_since(tp);
      }
    }
    const auto ts0 = hclock::now();
    CK(cudaStreamSynchronize(st));
    t_sync = us_since(ts0);
    const IterCtl* hc = reinterpret_cast<const IterCtl*>(ws.h_state + slot_bytes * kBatch);
    for (int j = 0; j < kBatch; ++j) {
      const IterState* hs_ = reinterpret_cast<const IterState*>(ws.h_state + slot_bytes * j);
      if (!hs_->valid) continue;
      const IterArrays harr = iter_arrays(const_cast<IterState*>(hs_), B);
      const int ncols = hs_->ncols, nrows = hs_->nrows;
      for (int s = 0; s < ncols; ++s) {
        run->step_kind.push_back(0);
        run->step_iter.push_back(k_host);
        run->step_index.push_back(harr.col_idx[s]);
        run->step_best.push_back(harr.col_best[s]);
        run->step_second.push_back(harr.col_second[s]);
      }
      for (int s = 0; s < nrows; ++s) {
        run->step_kind.push_back(1);
        run->step_iter.push_back(k_host);
        run->step_index.push_back(harr.row_idx[s]);
        run->step_best.push_back(harr.row_best[s]);
        run->step_second.push_back(harr.row_second[s]);
      }
      if (ncols == 0 || nrows == 0) break;  // ResidualExhausted: nothing committed
      const int width = hs_->width;
      for (int q = 0; q < width; ++q) {
        run->I.push_back(harr.row_idx[q]);
        run->J.push_back(harr.col_idx[q]);
      }
      run->block_start.push_back(r_host);
      run->block_width.push_back(width);
      r_host += width;
      itercur_iteration_record rec{};
      rec.k = k_host;
      rec.rho = hs_->rho;
      rec.cols_added = rec.rows_added = width;
      rec.col_truncated = 0;  // filled below from the requested block
      rec.row_truncated = nrows < ncols;
      rec.min_col_margin = min_margin(harr.col_best, harr.col_second, ncols);
      rec.min_row_margin = min_margin(harr.row_best, harr.row_second, nrows);
      const int64_t requested = std::min<int64_t>(b, max_rank - (r_host - width));
      rec.col_truncated = ncols < requested;
      run->iters.push_back(rec);
      ++k_host;
    }
    if (hc->r != r_host || hc->k != k_host) fail(ITERCUR_E_LOGIC, "device / host iteration bookkeeping diverged");
    if (cfg.observer && k_host > observed) {
      // driver.cpp:154: the observer sees the factors after the iteration (one per batch here)
      run->r = r_host;
      observed = k_host;
      cudaStream_t saved = g_alloc_stream;
      const int rc = cfg.observer(cfg.observer_user, run, &run->iters.back());
      g_alloc_stream = saved;
      CK(cudaSetDevice(run->device));
      if (rc != 0) fail(ITERCUR_E_RUNTIME, "iteration observer failed");
    }
    if (host_trace)
      fprintf(stderr, "[itercur batch] r=%lld capL=%lld grow=%.0fus capture=%.0fus launch=%.0fus sync=%.0fus total=%.0fus\n",
              static_cast<long long>(r_host), static_cast<long long>(run->capL), t_grow, t_capture, t_launch, t_sync,
              us_since(tb0));
    run->r = r_host;
    rho = hc->rho;
    done = hc->done != 0;
    if (done) {
      run->status = hc->status;
    } else if (r_host >= max_rank || k_host >= max_iters) {
      // the next iteration's begin would stop here with MaxRank (iter_begin_kernel): no need to
      // launch a batch of early-returning kernels to learn it (config 5: ~0.15 ms)
      done = true;
      run->status = ITERCUR_MAX_RANK;
    }
  }
  if (evs.on) {
    for (size_t q = 0; q < run->iters.size() && q < iter_events.size(); ++q) {
      const size_t e0 = iter_events[q];
      auto& rec = run->iters[q];
      rec.select_cols_s = elapsed_s(evs.get(e0), evs.get(e0 + 1));
      rec.row_residual_s = elapsed_s(evs.get(e0 + 1), evs.get(e0 + 2));
      rec.select_rows_s = elapsed_s(evs.get(e0 + 2), evs.get(e0 + 3));
      rec.core_s = elapsed_s(evs.get(e0 + 3), evs.get(e0 + 4));
      rec.downdate_s = elapsed_s(evs.get(e0 + 4), evs.get(e0 + 5));
    }
  }
  auto print_trace = [&](const char* name, const DevBuf<long long>& buf, int64_t k) {
    std::vector<long long> h(32 + 2 * 8192);
    CK(cudaMemcpyAsync(h.data(), buf.p, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fprintf(stderr,
            "[%s trace k=%lld] CTA0 cycles: main %lld exchange %lld fills %lld fwd %lld back %lld rt %lld "
            "dmma+y %lld norm %lld total %lld\n",
            name, static_cast<long long>(k), h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4],
            h[6] - h[5], h[7] - h[6], h[8] - h[7], h[8] - h[0]);
    std::vector<long long> starts, ends;
    for (int c = 0; c < 8192; ++c)
      if (h[32 + 2 * c]) {
        starts.push_back(h[32 + 2 * c]);
        ends.push_back(h[32 + 2 * c + 1]);
      }
    const int n = static_cast<int>(starts.size());
    if (n) {
      const long long t0 = *std::min_element(starts.begin(), starts.end());
      const long long t1 = *std::max_element(starts.begin(), starts.end());
      const long long e_fin = *std::max_element(ends.begin(), ends.end());
      std::vector<long long> dur(n);
      for (int c = 0; c < n; ++c) dur[c] = ends[c] - starts[c];
      std::sort(dur.begin(), dur.end());
      fprintf(stderr, "[%s trace] %d CTAs: last start +%lld ns, last end +%lld ns; CTA span ns min %lld median %lld max %lld\n",
              name, n, t1 - t0, e_fin - t0, dur[0], dur[n / 2], dur[n - 1]);
    }
  };
  if (ub_trace_env) print_trace("ub", ub_dbg, ub_trace_k);
  if (g1_trace_env) print_trace("g1", g1_dbg, g1_trace_k);
  run->final_rho = rho;
  run->total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  if (host_trace) fprintf(stderr, "[itercur done] total %.0fus\n", run->total_s * 1e6);
}

// ------------------------------------------------------------------ host input
// A host matrix to the device. Pinned (page-locked) memory goes straight to the copy engines.
// Pageable memory — the drop-in path: a numpy array handed to MatrixHandle.dense — would copy at
// ~11 GB/s through the driver's own bounce buffer (measured on the pool's B200 box, vs 55 GB/s
// pinned), so it is staged instead: column chunks copied by a pool of host threads into four
// pinned 64 MB buffers, each buffer's DMA overlapping the host copy of the next chunk.
class HostCopyPool {
 public:
  static HostCopyPool& get() {
    static HostCopyPool p;
    return p;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  // fn(t) for t in [0, size()), the caller runs t = 0
  void run(const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      pending_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostCopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const int n = static_cast<int>(std::max(1u, std::min(hw ? hw : 1u, 8u)));
    for (int t = 1; t < n; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~HostCopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void loop(int t) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = fn_;
      }
      (*fn)(t);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

bool host_is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// dst (m x n, ld m, device) <- src (m x n, ld lda, host), enqueued on st (returns after the last
// host copy; the DMA may still run)
void copy_host_matrix(double* dst, const double* src, int64_t m, int64_t n, int64_t lda, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  static const bool no_staging = env_flag("ITERCUR_NO_STAGED_H2D");
  if (no_staging || host_is_pinned(src)) {
    if (lda == m)
      CK(cudaMemcpyAsync(dst, src, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
    else
      CK(cudaMemcpy2DAsync(dst, sizeof(double) * m, src, sizeof(double) * lda, sizeof(double) * m, n,
                           cudaMemcpyHostToDevice, st));
    return;
  }
  constexpr int kBufs = 4;
  constexpr size_t kBufBytes = size_t(64) << 20;
  struct Staging {
    double* buf[kBufs] = {};
    cudaEvent_t ev[kBufs] = {};
    int device = -1;
  };
  thread_local Staging sg;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (sg.device != dev) {  // pinned buffers and events, once per thread and device
    for (int b = 0; b < kBufs; ++b) {
      if (sg.buf[b]) cudaFreeHost(sg.buf[b]);
      if (sg.ev[b]) cudaEventDestroy(sg.ev[b]);
      CK(cudaMallocHost(reinterpret_cast<void**>(&sg.buf[b]), kBufBytes));
      CK(cudaEventCreateWithFlags(&sg.ev[b], cudaEventDisableTiming));
    }
    sg.device = dev;
  }
  HostCopyPool& pool = HostCopyPool::get();
  const int64_t cols = std::max<int64_t>(1, static_cast<int64_t>(kBufBytes / sizeof(double)) / m);
  if (cols * m * static_cast<int64_t>(sizeof(double)) > static_cast<int64_t>(kBufBytes)) {
    // a single column larger than a staging buffer: the driver's path
    CK(cudaMemcpy2DAsync(dst, sizeof(double) * m, src, sizeof(double) * lda, sizeof(double) * m, n,
                         cudaMemcpyHostToDevice, st));
    return;
  }
  int64_t k = 0;
  for (int64_t j0 = 0; j0 < n; j0 += cols, ++k) {
    const int b = static_cast<int>(k % kBufs);
    const int64_t w = std::min(cols, n - j0);
    CK(cudaEventSynchronize(sg.ev[b]));  // that buffer's previous DMA (this call's or an earlier one's) is done
    double* stg = sg.buf[b];
    const int T = pool.size();
    const std::function<void(int)> part = [&](int t) {
      const int64_t total = w * m, per = (total + T - 1) / T;
      int64_t e = std::min(total, t * per);
      const int64_t end = std::min(total, e + per);
      while (e < end) {  // element e = (row e % m, column e / m) of the chunk
        const int64_t c = e / m, r = e % m, len = std::min(end - e, m - r);
        std::memcpy(stg + e, src + (j0 + c) * lda + r, sizeof(double) * len);
        e += len;
      }
    };
    pool.run(part);
    CK(cudaMemcpyAsync(dst + j0 * m, stg, sizeof(double) * w * m, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(sg.ev[b], st));
  }
}

// ------------------------------------------------------------------ exports
// Host entry: keep only C = A(:,J) and R^T = A(I,:)^T (r (m + n) doubles) and free the m x n
// device copy of A, so a live result does not pin the input's HBM (80 GB at configs 4/5).
void release_input_copy(itercur_run* run) {
  cudaStream_t st = run->wstream;
  g_alloc_stream = st;
  if (run->r > 0) {
    run->Cg.alloc(static_cast<size_t>(run->m) * run->r);
    run->RgT.alloc(static_cast<size_t>(run->n) * run->r);
    CK(launch_gather(run->A, 1, run->lda, run->m, run->dJ.p, nullptr, static_cast<int>(run->r), run->Cg.p, run->m, st));
    CK(launch_gather(run->A, run->lda, 1, run->n, run->dI.p, nullptr, static_cast<int>(run->r), run->RgT.p, run->n, st));
  }
  run->A_owned.reset();
  run->A = nullptr;
  CK(cudaStreamSynchronize(st));
}

// A rank of an NCCL-sharded run holds only its columns of A, Y and R~: exports that need the whole
// factors are collective operations it does not provide (indices, trace and the collective
// itercur_true_relative_error_sharded are available).
void require_whole_factors(const itercur_run* run, const char* what) {
  if (run->sh.active && run->sh.comm)
    fail(ITERCUR_E_LOGIC, std::string(what) + ": a rank of a column-sharded run holds only its shard's columns "
                                              "(use itercur_true_relative_error_sharded)");
}

void gather_host(const itercur_run* run, const double* src, int64_t row_stride, int64_t col_stride, int64_t K,
                 const int64_t* d_idx, int64_t w, double* out) {
  if (K == 0 || w == 0) return;
  DevBuf<double> tmp;
  tmp.alloc(static_cast<size_t>(K) * w);
  CK(launch_gather(src, row_stride, col_stride, K, d_idx, nullptr, static_cast<int>(w), tmp.p, K, run->stream));
  CK(cudaMemcpyAsync(out, tmp.p, sizeof(double) * K * w, cudaMemcpyDeviceToHost, run->stream));
  CK(cudaStreamSynchronize(run->stream));
}

// X^{-1} with X = A(I,J) = Lc * Uc, Lc = L(I,:) block-lower (diagonal blocks D_k),
// Uc = Rt(:,J) unit block-upper.  Zt = (Lc^{-1})^T by block forward substitution, then
// Xit = (Uc^{-1} Z)^T by block back substitution; core = Xit^T.
// Xit = X^{-T} (r x r, column-major, ld r) on the device, X = A(I, J).
void core_xit_device(const itercur_run* run, DevBuf<double>& Xit) {
  const int64_t r = run->r;
  cudaStream_t st = run->stream;
  const int B = static_cast<int>(run->bmax);
  DevBuf<double> Zt, T, Bg;
  Zt.alloc(static_cast<size_t>(r) * r);
  Xit.alloc(static_cast<size_t>(r) * r);
  T.alloc(static_cast<size_t>(r) * B);
  Bg.alloc(static_cast<size_t>(r) * B);
  DevBuf<int64_t> seq;
  {
    std::vector<int64_t> h(static_cast<size_t>(r));
    for (int64_t q = 0; q < r; ++q) h[q] = q;
    seq.alloc(r);
    CK(cudaMemcpyAsync(seq.p, h.data(), sizeof(int64_t) * r, cudaMemcpyHostToDevice, st));
  }
  const size_t nb = run->block_start.size();
  for (size_t kb = 0; kb < nb; ++kb) {
    const int64_t s = run->block_start[kb], w = run->block_width[kb];
    // Bg(k', q) = Lc(s+q, k') = L(I[s+q], k'), k' < s
    if (s > 0) CK(launch_gather(run->L.p, run->ldL, 1, s, run->dI.p + s, nullptr, static_cast<int>(w), Bg.p, s, st));
    TsGemmParams p;
    p.M = r;
    p.K = s;
    p.N = static_cast<int>(w);
    p.A = Zt.p;
    p.lda = r;
    p.B = Bg.p;
    p.bsk = 1;
    p.bsn = std::max<int64_t>(s, 1);
    p.base_mode = kBaseIdentityCols;
    p.col0 = s;
    p.alpha = -1.0;
    p.out_mode = kOutColMajor;
    p.C0 = T.p;
    p.ldc0 = r;
    CK(run_ts_gemm(p, st));
    CK(launch_rows_lu_solve(T.p, r, r, run->Dinv.p + run->bmax * s, run->bmax, nullptr, static_cast<int>(w),
                            Zt.p + r * s, r, st, nullptr, 0, run->Piv.p ? run->Piv.p + s : nullptr));
  }
  for (size_t kb = nb; kb-- > 0;) {
    const int64_t s = run->block_start[kb], w = run->block_width[kb];
    const int64_t e = s + w;
    // Bg(k', q) = Uc(s+q, e+k') = Rt(s+q, J[e+k'])
    if (r - e > 0) {
      CK(launch_gather2(run->Rt.p + run->ldR * s, run->ldR, run->dJ.p + e, r - e, static_cast<int>(w), Bg.p, r - e, st));
    }
    TsGemmParams p;
    p.M = r;
    p.K = r - e;
    p.N = static_cast<int>(w);
    p.A = Xit.p + r * e;
    p.lda = r;
    p.B = Bg.p;
    p.bsk = 1;
    p.bsn = std::max<int64_t>(r - e, 1);
    p.base_mode = kBaseContigCols;
    p.src = Zt.p;
    p.lds = r;
    p.col0 = s;
    p.alpha = -1.0;
    p.out_mode = kOutColMajor;
    p.C0 = Xit.p + r * s;
    p.ldc0 = r;
    CK(run_ts_gemm(p, st));
  }
}

void core_matrix_impl(const itercur_run* run, double* out) {
  const int64_t r = run->r;
  if (r == 0) return;
  cudaStream_t st = run->stream;
  DevBuf<double> Xit;
  core_xit_device(run, Xit);
  std::vector<double> h(static_cast<size_t>(r) * r);
  CK(cudaMemcpyAsync(h.data(), Xit.p, sizeof(double) * r * r, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  for (int64_t j = 0; j < r; ++j)
    for (int64_t i = 0; i < r; ++i) out[i + j * r] = h[j + i * r];  // core = Xit^T
}

// out = X^{-1} rhs (transposed = 0) or X^{-T} rhs (1): FactoredPinv::solve / solve_transposed
// (pinv.cpp:24-39) of the engine's exact core, on the device GEMM with the materialised inverse.
void core_apply_impl(const itercur_run* run, bool transposed, const double* rhs, int64_t k, int64_t ldr, double* out,
                     int64_t ldo) {
  const int64_t r = run->r;
  if (r == 0 || k == 0) return;
  cudaStream_t st = run->stream;
  DevBuf<double> Xit, op, B, C;
  core_xit_device(run, Xit);
  const int64_t ldop = even(r);
  op.alloc(static_cast<size_t>(ldop) * r);
  if (transposed) {  // X^{-T} = Xit
    CK(cudaMemcpy2DAsync(op.p, sizeof(double) * ldop, Xit.p, sizeof(double) * r, sizeof(double) * r, r,
                         cudaMemcpyDeviceToDevice, st));
  } else {  // X^{-1} = Xit^T
    CK(launch_transpose(Xit.p, r, r, r, op.p, ldop, st));
  }
  B.alloc(static_cast<size_t>(r) * k);
  C.alloc(static_cast<size_t>(r) * k);
  CK(cudaMemcpy2DAsync(B.p, sizeof(double) * r, rhs, sizeof(double) * ldr, sizeof(double) * r, k,
                       cudaMemcpyHostToDevice, st));
  constexpr int64_t kChunk = 1 << 20;  // columns per GEMM launch (grid.y bound)
  for (int64_t q0 = 0; q0 < k; q0 += kChunk) {
    TsGemmParams p;
    p.M = r;
    p.K = r;
    p.N = static_cast<int>(std::min(kChunk, k - q0));
    p.A = op.p;
    p.lda = ldop;
    p.B = B.p + q0 * r;
    p.bsk = 1;
    p.bsn = r;
    p.base_mode = kBaseNone;
    p.alpha = 1.0;
    p.out_mode = kOutColMajor;
    p.C0 = C.p + q0 * r;
    p.ldc0 = r;
    CK(run_ts_gemm(p, st));
  }
  CK(cudaMemcpy2DAsync(out, sizeof(double) * ldo, C.p, sizeof(double) * r, sizeof(double) * r, k,
                       cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

// ||A - L R~||_F^2 over columns [j0, j0 + w) of a device matrix Ap (column j0 at Ap, ld lda),
// summed into *d_out (fixed-order reduction).
void residual_sumsq_panel(const itercur_run* run, const double* Ap, int64_t lda, int64_t j0, int64_t w,
                          DevBuf<double>& part, double* d_out, cudaStream_t st) {
  TsGemmParams p;
  p.M = run->m;
  p.K = run->r;
  p.N = static_cast<int>(w);
  p.A = run->L.p;
  p.lda = run->ldL;
  p.B = run->Rt.p + j0;  // B(k, q) = R~(k, j0 + q)
  p.bsk = run->ldR;
  p.bsn = 1;
  p.base_mode = kBaseContigCols;
  p.src = Ap;
  p.lds = lda;
  p.col0 = 0;
  p.alpha = -1.0;
  p.out_mode = kOutNone;
  const int64_t parts = ts_gemm_grid_size(p.M, p.N);
  if (part.count < static_cast<size_t>(parts)) part.alloc(parts);
  p.norm_part = part.p;
  CK(run_ts_gemm(p, st));
  CK(launch_sum_partials(part.p, parts, d_out, st));
}

// true_relative_error(A, factors), proj/src/driver.cpp:169-190: ||A - C core R|| / ||A|| with
// C core R = L R~ (the incremental form). A is the run's own matrix or any m x n matrix given on
// the device or on the host (streamed through the device in column panels).
double true_error_impl(const itercur_run* run, const double* A, int64_t lda, bool on_device) {
  cudaStream_t st = run->stream;
  const int64_t m = run->m, n = run->n;
  if (on_device) {
    const double asq = device_sumsq(A, m, n, lda, st);
    const double a_norm = std::sqrt(asq);
    if (a_norm == 0.0) return 0.0;
    if (run->r == 0) return 1.0;
    DevBuf<double> part, outd;
    outd.alloc(1);
    constexpr int64_t kPanel = 1 << 30;
    double sq = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += kPanel) {
      residual_sumsq_panel(run, A + j0 * lda, lda, j0, std::min(kPanel, n - j0), part, outd.p, st);
      double h = 0.0;
      CK(cudaMemcpyAsync(&h, outd.p, sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      sq += h;
    }
    return std::sqrt(sq) / a_norm;
  }
  // host matrix: column panels of <= 512 MB through a device buffer; per-panel sums in panel order
  const int64_t w_max = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t(1) << 26) / std::max<int64_t>(m, 1)));
  const int64_t npanels = (n + w_max - 1) / w_max;
  DevBuf<double> panel, part, outd, apart;
  panel.alloc(static_cast<size_t>(m) * w_max);
  outd.alloc(2 * npanels);
  apart.alloc(148 * 8);
  for (int64_t pi = 0; pi < npanels; ++pi) {
    const int64_t j0 = pi * w_max, w = std::min(w_max, n - j0);
    CK(cudaMemcpy2DAsync(panel.p, sizeof(double) * m, A + j0 * lda, sizeof(double) * lda, sizeof(double) * m, w,
                         cudaMemcpyHostToDevice, st));
    CK(launch_sumsq(panel.p, m, w, m, apart.p, 148 * 8, outd.p + 2 * pi, st));
    if (run->r > 0) residual_sumsq_panel(run, panel.p, m, j0, w, part, outd.p + 2 * pi + 1, st);
  }
  std::vector<double> h(static_cast<size_t>(2 * npanels));
  CK(cudaMemcpyAsync(h.data(), outd.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double asq = 0.0, sq = 0.0;
  for (int64_t pi = 0; pi < npanels; ++pi) {
    asq += h[2 * pi];
    sq += h[2 * pi + 1];
  }
  const double a_norm = std::sqrt(asq);
  if (a_norm == 0.0) return 0.0;
  if (run->r == 0) return 1.0;
  return std::sqrt(sq) / a_norm;
}

// make_sketch(seed, b, A) + downdate_col_residual(estimator, factors) (proj/src/sketch.cpp:10-41)
// for a finished run's factors: rho = ||G A - G (C core R)|| / ||G A||. With the incremental
// form C core R = L R~, so G C core R = (G L) R~: the sketch operator is applied to L (m x r) by
// the same kernel, then Y^T -= R~^T (G L)^T on the engine's GEMM with ||Y||^2 fused.
double sketched_residual_impl(const itercur_run* run, const double* A, int64_t lda, int64_t b, uint64_t seed,
                              int32_t kind, int32_t sparse_nnz) {
  cudaStream_t st = run->stream;
  const int64_t m = run->m, n = run->n;
  if (b < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "block size must be at least 1");
  if (b > m) fail(ITERCUR_E_INVALID_ARGUMENT, "block exceeds row count");
  const int64_t c = sketch_rows(b), cp = round_up(c, 8);
  const int k = kind == ITERCUR_SKETCH_SPARSE_SIGN ? kSketchSparseSign : kSketchGaussian;
  DevBuf<double> Y, GL, scal, part, outd;
  SketchBuffers sb;
  Y.alloc(static_cast<size_t>(cp) * n);
  scal.alloc(4);
  const int64_t r = run->r;
  apply_sketch(A, m, n, lda, k, sparse_nnz, seed, kStreamSketch, c, cp, Y.p, SketchStats{scal.p, scal.p + 1},
               sb, st);
  double h[2];
  CK(cudaMemcpyAsync(h, scal.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double ga_norm = std::sqrt(h[1]);
  if (r == 0 || ga_norm == 0.0) return ga_norm > 0.0 ? 1.0 : 0.0;  // sketch.cpp:27-30
  GL.alloc(static_cast<size_t>(cp) * r);
  // the same operator on L (the dense operator, if any, is reused)
  apply_sketch(run->L.p, m, r, run->ldL, k, sparse_nnz, seed, kStreamSketch, c, cp, GL.p,
               SketchStats{scal.p + 2, scal.p + 3}, sb, st, nullptr, sb.S.p != nullptr);
  TsGemmParams p;
  p.M = n;
  p.K = r;
  p.N = static_cast<int>(c);
  p.A = run->Rt.p;  // R~^T (n x r), column-major with ld ldR
  p.lda = run->ldR;
  p.B = GL.p;       // B(q, h) = (G L)(h, q)
  p.bsk = cp;
  p.bsn = 1;
  p.base_mode = kBaseInPlaceRowMajor;
  p.C0 = Y.p;       // Y^T(j, h) = Y[h + j * cp]
  p.ldc0 = cp;
  p.out_mode = kOutRowMajor;
  p.alpha = -1.0;
  const int64_t parts = ts_gemm_grid_size(p.M, p.N);
  part.alloc(parts);
  outd.alloc(1);
  p.norm_part = part.p;
  CK(run_ts_gemm(p, st));
  CK(launch_sum_partials(part.p, parts, outd.p, st));
  double ysq = 0.0;
  CK(cudaMemcpyAsync(&ysq, outd.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return std::sqrt(ysq) / ga_norm;
}

void require_device() {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    fail(ITERCUR_E_CUDA, "no CUDA device: the B200 engine has no CPU fallback");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) fail(ITERCUR_E_CUDA, "the B200 engine requires an sm_100 device");
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

void itercur_config_default(itercur_config* cfg) { *cfg = default_config(); }
const char* itercur_last_error(void) { return g_last_error.c_str(); }
int itercur_abi_version(void) { return ITERCUR_B200_ABI_VERSION; }

// Load every kernel of the engine's modules now (CUDA lazy loading would otherwise load each on its
// first launch, inside the first iterative_cur call): one representative kernel per translation
// unit gives its module; the driver enumerates and loads the module's functions.
int itercur_preload(int32_t* functions_loaded) {
  return guarded([&] {
    require_device();
    using FnGetModule = CUresult (*)(CUmodule*, CUfunction);
    using FnCount = CUresult (*)(unsigned int*, CUmodule);
    using FnEnum = CUresult (*)(CUfunction*, unsigned int, CUmodule);
    using FnLoad = CUresult (*)(CUfunction);
    auto entry = [](const char* name, int ver) -> void* {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPointByVersion(name, &p, ver, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        return nullptr;
      return p;
    };
    auto get_module = reinterpret_cast<FnGetModule>(entry("cuFuncGetModule", 11000));
    auto count_fns = reinterpret_cast<FnCount>(entry("cuModuleGetFunctionCount", 12040));
    auto enum_fns = reinterpret_cast<FnEnum>(entry("cuModuleEnumerateFunctions", 12040));
    auto load_fn = reinterpret_cast<FnLoad>(entry("cuFuncLoad", 12040));
    int32_t loaded = 0;
    const void* anchors[] = {module_anchor_gemm(), module_anchor_lupp(), module_anchor_misc(),
                             module_anchor_qrcp(), module_anchor_shard(), module_anchor_sketch()};
    for (const void* k : anchors) {
      cudaFunction_t f = nullptr;
      if (cudaGetFuncBySymbol(&f, k) != cudaSuccess) continue;
      if (!get_module || !count_fns || !enum_fns || !load_fn) {  // older driver: the anchor alone
        cudaFuncAttributes attr;
        if (cudaFuncGetAttributes(&attr, k) == cudaSuccess) ++loaded;
        continue;
      }
      CUmodule mod = nullptr;
      unsigned int nf = 0;
      if (get_module(&mod, reinterpret_cast<CUfunction>(f)) != CUDA_SUCCESS || count_fns(&nf, mod) != CUDA_SUCCESS)
        continue;
      std::vector<CUfunction> fns(nf);
      if (nf == 0 || enum_fns(fns.data(), nf, mod) != CUDA_SUCCESS) continue;
      for (CUfunction fn : fns)
        if (load_fn(fn) == CUDA_SUCCESS) ++loaded;
    }
    cudaGetLastError();
    if (functions_loaded) *functions_loaded = loaded;
  });
}

int itercur_iterative_cur_device(const double* dA, int64_t m, int64_t n, int64_t lda, const itercur_config* cfg,
                                 void* stream, itercur_run** out) {
  *out = nullptr;
  return guarded([&] {
    require_device();
    auto run = std::make_unique<itercur_run>();
    CK(cudaGetDevice(&run->device));
    run->stream = static_cast<cudaStream_t>(stream);
    run->wstream = work_stream();
    {  // the work stream starts after everything already queued on the caller's stream
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CK(cudaEventRecord(ev, run->stream));
      CK(cudaStreamWaitEvent(run->wstream, ev, 0));
      cudaEventDestroy(ev);
    }
    run->m = m;
    run->n = n;
    run->lda = lda;
    run->A = dA;
    run->cfg = cfg ? *cfg : default_config();
    configure_mempool_once();
    g_alloc_stream = run->wstream;
    run_iterative_cur(run.get());
    *out = run.release();
  });
}

int itercur_shard_range(int64_t n_total, int32_t world, int32_t rank, int64_t* offset, int64_t* count) {
  return guarded([&] {
    if (n_total < 1 || world < 1 || rank < 0 || rank >= world)
      fail(ITERCUR_E_INVALID_ARGUMENT, "shard_range: invalid arguments");
    const int64_t blk = shard_block(n_total, world);
    const int64_t off = std::min<int64_t>(n_total, static_cast<int64_t>(rank) * blk);
    *offset = off;
    *count = std::min<int64_t>(blk, n_total - off);
  });
}

namespace {
void start_run(itercur_run* run, const double* dA, int64_t m, int64_t n, int64_t lda, const itercur_config* cfg,
               void* stream) {
  CK(cudaGetDevice(&run->device));
  run->stream = static_cast<cudaStream_t>(stream);
  run->wstream = work_stream();
  {  // the work stream starts after everything already queued on the caller's stream
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, run->stream));
    CK(cudaStreamWaitEvent(run->wstream, ev, 0));
    cudaEventDestroy(ev);
  }
  run->m = m;
  run->n = n;
  run->lda = lda;
  run->A = dA;
  run->cfg = cfg ? *cfg : default_config();
  configure_mempool_once();
  g_alloc_stream = run->wstream;
}
}  // namespace

int itercur_iterative_cur_sharded_device(const double* dA, int64_t m, int64_t n_local, int64_t lda, int64_t n_total,
                                         const itercur_config* cfg, void* comm, void* stream, itercur_run** out) {
  *out = nullptr;
  return guarded([&] {
    require_device();
    const NcclApi* nc = nccl_api();
    if (!nc) fail(ITERCUR_E_CUDA, std::string("NCCL unavailable: ") + nccl_load_error());
    if (!comm) fail(ITERCUR_E_INVALID_ARGUMENT, "sharded run: null communicator");
    auto run = std::make_unique<itercur_run>();
    ShardSpec& sh = run->sh;
    sh.active = true;
    sh.comm = static_cast<ncclComm_t>(comm);
    if (nc->CommCount(sh.comm, &sh.world) != ncclSuccess || nc->CommUserRank(sh.comm, &sh.rank) != ncclSuccess)
      fail(ITERCUR_E_CUDA, "sharded run: cannot query the communicator");
    if (n_total < 2 * sh.world) fail(ITERCUR_E_INVALID_ARGUMENT, "sharded run: fewer than 2 columns per rank");
    const int64_t blk = shard_block(n_total, sh.world);
    const int64_t off = std::min<int64_t>(n_total, static_cast<int64_t>(sh.rank) * blk);
    if (n_local != std::min<int64_t>(blk, n_total - off) || n_local < 1)
      fail(ITERCUR_E_INVALID_ARGUMENT, "sharded run: this rank's block must be columns [" + std::to_string(off) + ", " +
                                           std::to_string(off + std::min<int64_t>(blk, n_total - off)) +
                                           ") (itercur_shard_range)");
    sh.nloc = 1;
    sh.n_total = n_total;
    sh.goff.assign(1, off);
    sh.cnt.assign(1, n_local);
    start_run(run.get(), dA, m, n_local, lda, cfg, stream);
    if (run->cfg.observer) fail(ITERCUR_E_INVALID_ARGUMENT, "sharded run: no iteration observer");
    run_iterative_cur(run.get());
    *out = run.release();
  });
}

int itercur_iterative_cur_sharded_emulated(const double* dA, int64_t m, int64_t n, int64_t lda, int32_t shards,
                                           const itercur_config* cfg, void* stream, itercur_run** out) {
  *out = nullptr;
  return guarded([&] {
    require_device();
    if (shards < 1 || n < 2 * static_cast<int64_t>(shards))
      fail(ITERCUR_E_INVALID_ARGUMENT, "sharded run: fewer than 2 columns per shard");
    auto run = std::make_unique<itercur_run>();
    ShardSpec& sh = run->sh;
    sh.active = true;
    sh.nloc = shards;
    sh.n_total = n;
    const int64_t blk = shard_block(n, shards);
    for (int s = 0; s < shards; ++s) {
      const int64_t off = std::min<int64_t>(n, s * blk);
      sh.goff.push_back(off);
      sh.cnt.push_back(std::min<int64_t>(blk, n - off));
      if (sh.cnt.back() < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "sharded run: an empty shard");
    }
    start_run(run.get(), dA, m, n, lda, cfg, stream);
    run_iterative_cur(run.get());
    *out = run.release();
  });
}

int itercur_true_relative_error_sharded(const itercur_run* run, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    if (!(run->sh.active && run->sh.comm)) {  // the whole factors are local
      if (!run->A) fail(ITERCUR_E_LOGIC, "the run released its device copy of A");
      *out = true_error_impl(run, run->A, run->lda, true);
      return;
    }
    // this rank's ||A_s||^2 and ||A_s - L R~_s||^2, summed over the ranks (driver.cpp:169-190)
    cudaStream_t st = run->stream;
    const NcclApi* nc = nccl_api();
    DevBuf<double> part, outd;
    outd.alloc(2);
    DevBuf<double> apart;
    apart.alloc(148 * 8);
    CK(launch_sumsq(run->A, run->m, run->n, run->lda, apart.p, 148 * 8, outd.p, st));
    if (run->r > 0) {
      residual_sumsq_panel(run, run->A, run->lda, 0, run->n, part, outd.p + 1, st);
    } else {
      CK(cudaMemsetAsync(outd.p + 1, 0, sizeof(double), st));
    }
    if (nc->AllReduce(outd.p, outd.p, 2, ncclDouble, ncclSum, run->sh.comm, st) != ncclSuccess)
      fail(ITERCUR_E_CUDA, "NCCL allreduce failed (true_relative_error_sharded)");
    double h[2];
    CK(cudaMemcpyAsync(h, outd.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const double a_norm = std::sqrt(h[0]);
    *out = a_norm == 0.0 ? 0.0 : (run->r == 0 ? 1.0 : std::sqrt(h[1]) / a_norm);
  });
}

int itercur_nccl_unique_id(void* id_out) {
  return guarded([&] {
    const NcclApi* nc = nccl_api();
    if (!nc) fail(ITERCUR_E_CUDA, std::string("NCCL unavailable: ") + nccl_load_error());
    ncclUniqueId id;
    if (nc->GetUniqueId(&id) != ncclSuccess) fail(ITERCUR_E_CUDA, "ncclGetUniqueId failed");
    std::memcpy(id_out, &id, sizeof(id));
  });
}
int itercur_nccl_comm_init(int32_t world, const void* id_in, int32_t rank, void** comm_out) {
  *comm_out = nullptr;
  return guarded([&] {
    require_device();
    const NcclApi* nc = nccl_api();
    if (!nc) fail(ITERCUR_E_CUDA, std::string("NCCL unavailable: ") + nccl_load_error());
    ncclUniqueId id;
    std::memcpy(&id, id_in, sizeof(id));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = nc->CommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) fail(ITERCUR_E_CUDA, std::string("ncclCommInitRank: ") + nc->GetErrorString(r));
    *comm_out = comm;
  });
}
int itercur_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    const NcclApi* nc = nccl_api();
    if (nc && comm) nc->CommDestroy(static_cast<ncclComm_t>(comm));
  });
}

int itercur_iterative_cur_host(const double* A, int64_t m, int64_t n, int64_t lda, const itercur_config* cfg,
                               itercur_run** out) {
  *out = nullptr;
  return guarded([&] {
    require_device();
    auto run = std::make_unique<itercur_run>();
    CK(cudaGetDevice(&run->device));
    run->stream = nullptr;
    run->wstream = work_stream();
    configure_mempool_once();
    g_alloc_stream = run->wstream;
    run->m = m;
    run->n = n;
    run->lda = std::max<int64_t>(m, 1);
    if (m > 0 && n > 0) {
      static const bool trace = env_flag("ITERCUR_HOST_TRACE");
      const auto t0 = std::chrono::steady_clock::now();
      run->A_owned.alloc(static_cast<size_t>(m) * n);
      const auto t1 = std::chrono::steady_clock::now();
      copy_host_matrix(run->A_owned.p, A, m, n, lda, run->wstream);
      if (trace) {
        CK(cudaStreamSynchronize(run->wstream));
        const auto t2 = std::chrono::steady_clock::now();
        fprintf(stderr, "[itercur host entry] alloc %.1f ms, H2D %.1f ms (%.1f GB/s)\n",
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count(),
                8.0 * m * n / std::chrono::duration<double>(t2 - t1).count() / 1e9);
      }
      run->A = run->A_owned.p;
    }
    run->cfg = cfg ? *cfg : default_config();
    const auto tr0 = std::chrono::steady_clock::now();
    run_iterative_cur(run.get());
    const auto tr1 = std::chrono::steady_clock::now();
    if (!run->cfg.keep_device_copy && run->A_owned.p) release_input_copy(run.get());
    if (env_flag("ITERCUR_HOST_TRACE"))
      fprintf(stderr, "[itercur host entry] run %.1f ms, release %.1f ms\n",
              std::chrono::duration<double, std::milli>(tr1 - tr0).count(),
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tr1).count());
    *out = run.release();
  });
}

int64_t itercur_run_rank(const itercur_run* run) { return run ? run->r : 0; }
int64_t itercur_run_rows(const itercur_run* run) { return run ? run->m : 0; }
int64_t itercur_run_cols(const itercur_run* run) { return run ? run->n : 0; }
int itercur_run_indices(const itercur_run* run, int64_t* row_indices, int64_t* col_indices) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    if (row_indices) std::copy(run->I.begin(), run->I.end(), row_indices);
    if (col_indices) std::copy(run->J.begin(), run->J.end(), col_indices);
  });
}
int32_t itercur_run_status(const itercur_run* run) { return run ? run->status : ITERCUR_CONVERGED; }
double itercur_run_final_rho(const itercur_run* run) { return run ? run->final_rho : 1.0; }
double itercur_run_threshold(const itercur_run* run) { return run ? run->threshold : 0.0; }
double itercur_run_sketch_seconds(const itercur_run* run) { return run ? run->sketch_s : 0.0; }
double itercur_run_total_seconds(const itercur_run* run) { return run ? run->total_s : 0.0; }
double itercur_run_ga_norm(const itercur_run* run) { return run ? run->ga_norm : 0.0; }
const char* itercur_run_note(const itercur_run* run) { return run ? run->note.c_str() : ""; }
int64_t itercur_run_num_iterations(const itercur_run* run) { return run ? static_cast<int64_t>(run->iters.size()) : 0; }
int itercur_run_iterations(const itercur_run* run, itercur_iteration_record* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    std::copy(run->iters.begin(), run->iters.end(), out);
  });
}
int64_t itercur_run_kernel_launches(const itercur_run* run) { return run ? run->launches : 0; }
int64_t itercur_run_num_steps(const itercur_run* run) { return run ? static_cast<int64_t>(run->step_index.size()) : 0; }
int itercur_run_steps(const itercur_run* run, int32_t* kind, int64_t* iter, int64_t* index, double* best,
                      double* second) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    std::copy(run->step_kind.begin(), run->step_kind.end(), kind);
    std::copy(run->step_iter.begin(), run->step_iter.end(), iter);
    std::copy(run->step_index.begin(), run->step_index.end(), index);
    std::copy(run->step_best.begin(), run->step_best.end(), best);
    std::copy(run->step_second.begin(), run->step_second.end(), second);
  });
}
int itercur_run_c_matrix(const itercur_run* run, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    require_whole_factors(run, "c_matrix");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    // C(i, q) = A(i, J[q]): out(k=i, q) = A[i * 1 + J[q] * lda]
    if (run->A) {
      gather_host(run, run->A, 1, run->lda, run->m, run->dJ.p, run->r, out);
    } else if (run->r > 0) {
      CK(cudaMemcpyAsync(out, run->Cg.p, sizeof(double) * run->m * run->r, cudaMemcpyDeviceToHost, run->stream));
      CK(cudaStreamSynchronize(run->stream));
    }
  });
}
int itercur_run_r_matrix(const itercur_run* run, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    require_whole_factors(run, "r_matrix");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    // R^T(j, q) = A(I[q], j): gathered as (n x r), then transposed on the host
    std::vector<double> t(static_cast<size_t>(run->n) * run->r);
    if (run->A) {
      gather_host(run, run->A, run->lda, 1, run->n, run->dI.p, run->r, t.data());
    } else if (run->r > 0) {
      CK(cudaMemcpyAsync(t.data(), run->RgT.p, sizeof(double) * t.size(), cudaMemcpyDeviceToHost, run->stream));
      CK(cudaStreamSynchronize(run->stream));
    }
    for (int64_t q = 0; q < run->r; ++q)
      for (int64_t j = 0; j < run->n; ++j) out[q + j * run->r] = t[j + q * run->n];
  });
}
int itercur_run_core_matrix(const itercur_run* run, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    require_whole_factors(run, "core_matrix");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    core_matrix_impl(run, out);
  });
}
int itercur_true_relative_error_device(const itercur_run* run, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    require_whole_factors(run, "true_relative_error");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    if (!run->A)
      fail(ITERCUR_E_LOGIC, "the run released its device copy of A (host entry): pass the matrix to "
                            "itercur_true_relative_error_matrix");
    *out = true_error_impl(run, run->A, run->lda, true);
  });
}
int itercur_true_relative_error_matrix(const itercur_run* run, const double* A, int64_t m, int64_t n, int64_t lda,
                                       int32_t a_on_device, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    require_whole_factors(run, "true_relative_error");
    if (m != run->m || n != run->n)
      fail(ITERCUR_E_INVALID_ARGUMENT, "true_relative_error: matrix is " + std::to_string(m) + "x" +
                                           std::to_string(n) + ", factors are for " + std::to_string(run->m) + "x" +
                                           std::to_string(run->n));
    if (lda < std::max<int64_t>(m, 1)) fail(ITERCUR_E_INVALID_ARGUMENT, "true_relative_error: lda < rows");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    *out = true_error_impl(run, A, lda, a_on_device != 0);
  });
}
int itercur_run_core_apply(const itercur_run* run, int32_t transposed, const double* rhs, int64_t k, int64_t ldr,
                           double* out, int64_t ldo) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    require_whole_factors(run, "core_apply");
    if (k < 0 || ldr < std::max<int64_t>(run->r, 1) || ldo < std::max<int64_t>(run->r, 1))
      fail(ITERCUR_E_INVALID_ARGUMENT, "core_apply: invalid shape");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    core_apply_impl(run, transposed != 0, rhs, k, ldr, out, ldo);
  });
}
int itercur_sketched_residual_device(const itercur_run* run, int64_t b, uint64_t seed, int32_t kind,
                                     int32_t sparse_nnz, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    require_whole_factors(run, "sketched_residual");
    if (!run->A)
      fail(ITERCUR_E_LOGIC, "the run released its device copy of A (host entry): pass the matrix to "
                            "itercur_sketched_residual_matrix");
    *out = sketched_residual_impl(run, run->A, run->lda, b, seed, kind, sparse_nnz);
  });
}
int itercur_sketched_residual_matrix(const itercur_run* run, const double* dA, int64_t lda, int64_t b, uint64_t seed,
                                     int32_t kind, int32_t sparse_nnz, double* out) {
  return guarded([&] {
    if (!run) fail(ITERCUR_E_LOGIC, "null run");
    require_whole_factors(run, "sketched_residual");
    if (!dA || lda < std::max<int64_t>(run->m, 1)) fail(ITERCUR_E_INVALID_ARGUMENT, "sketched residual: invalid matrix");
    CK(cudaSetDevice(run->device));
    g_alloc_stream = run->stream;
    *out = sketched_residual_impl(run, dA, lda, b, seed, kind, sparse_nnz);
  });
}
int32_t itercur_run_holds_matrix(const itercur_run* run) { return run && run->A ? 1 : 0; }
int itercur_copy_to_host(void* dst, const void* d_src, uint64_t bytes) {
  return guarded([&] {
    require_device();
    if (bytes) CK(cudaMemcpy(dst, d_src, bytes, cudaMemcpyDeviceToHost));
  });
}
int itercur_fro_norm_device(const double* dA, int64_t m, int64_t n, int64_t lda, void* stream, double* out) {
  return guarded([&] {
    require_device();
    if (m < 0 || n < 0 || (m > 0 && n > 0 && lda < m)) fail(ITERCUR_E_INVALID_ARGUMENT, "fro_norm: invalid shape");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    g_alloc_stream = st;
    *out = (m == 0 || n == 0) ? 0.0 : std::sqrt(device_sumsq(dA, m, n, lda, st));
  });
}
void itercur_run_free(itercur_run* run) { delete run; }

int itercur_fro_norm_host(const double* A, int64_t m, int64_t n, int64_t lda, double* out) {
  return guarded([&] {
    require_device();
    if (m < 0 || n < 0 || (m > 0 && n > 0 && lda < m)) fail(ITERCUR_E_INVALID_ARGUMENT, "fro_norm: invalid shape");
    if (m == 0 || n == 0) {
      *out = 0.0;
      return;
    }
    cudaStream_t st = work_stream();
    configure_mempool_once();
    g_alloc_stream = st;
    // column panels of <= 512 MB through the device; per-panel sums added in panel order
    const int64_t w_max = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t(1) << 26) / m));
    DevBuf<double> panel;
    panel.alloc(static_cast<size_t>(m) * w_max);
    double sq = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += w_max) {
      const int64_t w = std::min(w_max, n - j0);
      copy_host_matrix(panel.p, A + j0 * lda, m, w, lda, st);
      sq += device_sumsq(panel.p, m, w, m, st);
    }
    *out = std::sqrt(sq);
  });
}

int itercur_dense_apply_host(const double* X, int64_t r, int32_t transposed, const double* rhs, int64_t k,
                             double* out) {
  return guarded([&] {
    require_device();
    if (r < 0 || k < 0) fail(ITERCUR_E_INVALID_ARGUMENT, "dense_apply: invalid shape");
    if (r == 0 || k == 0) return;
    cudaStream_t st = work_stream();
    configure_mempool_once();
    g_alloc_stream = st;
    const int64_t ldop = even(r);
    DevBuf<double> Xd, op, B, C;
    Xd.alloc(static_cast<size_t>(r) * r);
    op.alloc(static_cast<size_t>(ldop) * r);
    B.alloc(static_cast<size_t>(r) * k);
    C.alloc(static_cast<size_t>(r) * k);
    CK(cudaMemcpyAsync(Xd.p, X, sizeof(double) * r * r, cudaMemcpyHostToDevice, st));
    if (transposed)
      CK(launch_transpose(Xd.p, r, r, r, op.p, ldop, st));
    else
      CK(cudaMemcpy2DAsync(op.p, sizeof(double) * ldop, Xd.p, sizeof(double) * r, sizeof(double) * r, r,
                           cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(B.p, rhs, sizeof(double) * r * k, cudaMemcpyHostToDevice, st));
    constexpr int64_t kChunk = 1 << 20;
    for (int64_t q0 = 0; q0 < k; q0 += kChunk) {
      TsGemmParams p;
      p.M = r;
      p.K = r;
      p.N = static_cast<int>(std::min(kChunk, k - q0));
      p.A = op.p;
      p.lda = ldop;
      p.B = B.p + q0 * r;
      p.bsk = 1;
      p.bsn = r;
      p.base_mode = kBaseNone;
      p.alpha = 1.0;
      p.out_mode = kOutColMajor;
      p.C0 = C.p + q0 * r;
      p.ldc0 = r;
      CK(run_ts_gemm(p, st));
    }
    CK(cudaMemcpyAsync(out, C.p, sizeof(double) * r * k, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int itercur_adjusted_threshold(double epsilon, double delta, double alpha, int64_t c, double* out) {
  return guarded([&] { *out = adjusted_threshold_impl(epsilon, delta, alpha, c); });
}
int itercur_gratton_tail(int64_t c, double tau, double* out) {
  return guarded([&] { *out = gratton_tail_impl(c, tau); });
}
int64_t itercur_sketch_rows_for_block(int64_t b) { return sketch_rows(b); }

int itercur_gaussian_matrix_device(int64_t rows, int64_t cols, uint64_t seed, uint32_t stream_tag, double* dOut,
                                   void* stream) {
  return guarded([&] {
    require_device();
    CK(launch_gaussian_matrix(rows, cols, seed, stream_tag, dOut, static_cast<cudaStream_t>(stream)));
    CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  });
}

int itercur_sketch_device(const double* dA, int64_t m, int64_t n, int64_t lda, int64_t b, uint64_t seed, int32_t kind,
                          int32_t sparse_nnz, double* dY, double* ga_norm, double* a_norm, void* stream) {
  return guarded([&] {
    require_device();
    // make_sketch validation, proj/src/sketch.cpp:11-13
    if (b < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "block size must be at least 1");
    if (m == 0 || n == 0) fail(ITERCUR_E_INVALID_ARGUMENT, "matrix must be nonempty");
    if (b > m) fail(ITERCUR_E_INVALID_ARGUMENT, "block exceeds row count");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    configure_mempool_once();
    g_alloc_stream = st;
    const int64_t c = sketch_rows(b), cp = round_up(c, 8);
    DevBuf<double> Yp, scal;
    SketchBuffers sb;
    Yp.alloc(static_cast<size_t>(cp) * n);
    scal.alloc(2);
    const int k = kind == ITERCUR_SKETCH_SPARSE_SIGN ? kSketchSparseSign : kSketchGaussian;
    SketchStats stats{scal.p, scal.p + 1};
    apply_sketch(dA, m, n, lda, k, sparse_nnz, seed, kStreamSketch, c, cp, Yp.p, stats, sb, st);
    // compact to ld = c
    CK(cudaMemcpy2DAsync(dY, sizeof(double) * c, Yp.p, sizeof(double) * cp, sizeof(double) * c, n,
                         cudaMemcpyDeviceToDevice, st));
    double h[2];
    CK(cudaMemcpyAsync(h, scal.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (a_norm) *a_norm = std::sqrt(h[0]);
    if (ga_norm) *ga_norm = std::sqrt(h[1]);
  });
}

static int select_impl(const double* dM, int64_t rows, int64_t cols, int64_t ldm, int64_t b, int32_t is_columns,
                       double pivot_floor, const int64_t* exclude, int64_t n_exclude, int64_t* idx_out, int64_t* n_idx,
                       int32_t* truncated, double* last_pivot, double* best_out, double* second_out, void* stream,
                       int32_t method) {
  return guarded([&] {
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    configure_mempool_once();
    g_alloc_stream = st;
    // select.cpp:24-28, 124-126, 143
    if (!(pivot_floor > 0.0 && pivot_floor < 1.0)) fail(ITERCUR_E_INVALID_ARGUMENT, "pivot_floor must lie in (0, 1)");
    if (is_columns && (b < 0 || b > rows))
      fail(ITERCUR_E_INVALID_ARGUMENT, "select_columns: block size " + std::to_string(b) + " exceeds sketch rows " +
                                           std::to_string(rows));
    if (!is_columns && b < 0) fail(ITERCUR_E_INVALID_ARGUMENT, "select_rows: negative block size");
    // LUPP works on W = M^T (columns) or M (rows); candidates are W's rows
    const int64_t wrows = is_columns ? cols : rows;
    const int64_t wcols = is_columns ? rows : cols;
    const int64_t steps = std::min<int64_t>(is_columns ? b : std::min(b, cols), wcols);
    std::vector<uint8_t> hmask(static_cast<size_t>(std::max<int64_t>(wrows, 1)), 0);
    for (int64_t q = 0; q < n_exclude; ++q) {
      const int64_t e = exclude[q];
      if (e < 0 || e >= wrows)
        fail(ITERCUR_E_OUT_OF_RANGE, std::string(is_columns ? "select_columns" : "select_rows") +
                                         ": excluded index " + std::to_string(e) + " out of range");
      hmask[e] = 1;
    }
    if (rows * cols > 0) {
      const unsigned long long zero = 0;
      (void)zero;
      DevBuf<unsigned long long> cnt;
      cnt.alloc(1);
      CK(launch_count_nonfinite(dM, rows, cols, ldm, cnt.p, st));
      unsigned long long h = 0;
      CK(cudaMemcpyAsync(&h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (h) fail(ITERCUR_E_INVALID_ARGUMENT, "selection input must be finite");
    }
    *n_idx = 0;
    *last_pivot = 0.0;
    if (steps <= 0 || wrows == 0) {
      *truncated = (0 < b) ? 1 : 0;
      return;
    }
    DevBuf<double> W, scal;
    DevBuf<uint8_t> mask;
    DevBuf<char> scratch, outs;
    const int64_t ldw = even(wrows);
    const bool qrcp = method == ITERCUR_PIVOT_QRCP;
    const int64_t ldq = even(rows);  // QRCP works on a copy of M itself
    W.alloc(qrcp ? static_cast<size_t>(ldq) * cols : static_cast<size_t>(ldw) * steps);
    if (qrcp)
      CK(cudaMemcpy2DAsync(W.p, sizeof(double) * ldq, dM, sizeof(double) * ldm, sizeof(double) * rows, cols,
                           cudaMemcpyDeviceToDevice, st));
    else if (is_columns)
      CK(launch_transpose_rows(dM, ldm, cols, static_cast<int>(steps), W.p, ldw, st));
    else
      CK(cudaMemcpy2DAsync(W.p, sizeof(double) * ldw, dM, sizeof(double) * ldm, sizeof(double) * rows, steps,
                           cudaMemcpyDeviceToDevice, st));
    scal.alloc(1);
    DevBuf<double> part;
    part.alloc(148 * 8);
    CK(launch_sumsq(dM, rows, cols, ldm, part.p, 148 * 8, scal.p, st));
    mask.alloc(wrows);
    CK(cudaMemcpyAsync(mask.p, hmask.data(), wrows, cudaMemcpyHostToDevice, st));
    scratch.alloc(lupp_scratch_bytes(static_cast<int>(steps)));
    CK(lupp_scratch_init(scratch.p, st));
    const int S = static_cast<int>(steps);
    outs.alloc(sizeof(int64_t) * S * 3 + 16);
    int64_t* d_idx = reinterpret_cast<int64_t*>(outs.p);
    double* d_best = reinterpret_cast<double*>(d_idx + S);
    double* d_second = d_best + S;
    int* d_count = reinterpret_cast<int*>(d_second + S);
    LuppArgs la{};
    la.W = W.p;
    la.rows = wrows;
    la.ldw = ldw;
    la.cols_max = S;
    la.mask = mask.p;
    la.epoch = 2;
    la.d_norm_sq = scal.p;
    la.pivot_floor = pivot_floor;
    la.d_idx = d_idx;
    la.d_best = d_best;
    la.d_second = d_second;
    la.d_count = d_count;
    if (qrcp) {  // candidates: columns of M (select_columns) or rows of M (select_rows)
      DevBuf<char> qs;
      qs.alloc(qrcp_scratch_bytes());
      CK(run_qrcp(W.p, wrows, static_cast<int>(wcols), nullptr, is_columns ? 1 : ldq, is_columns ? ldq : 1, nullptr, S,
                  mask.p, 2, scal.p, pivot_floor, d_idx, d_best, d_second, d_count, nullptr, nullptr, qs.p, nullptr,
                  st));
      CK(cudaStreamSynchronize(st));
    } else {
      CK(run_lupp_with_scratch(la, scratch.p, st, nullptr));
    }
    std::vector<char> h(outs.count);
    CK(cudaMemcpyAsync(h.data(), outs.p, outs.count, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t* hi = reinterpret_cast<const int64_t*>(h.data());
    const double* hb = reinterpret_cast<const double*>(hi + S);
    const double* hsd = hb + S;
    const int cnt = *reinterpret_cast<const int*>(hsd + S);
    *n_idx = cnt;
    for (int q = 0; q < cnt; ++q) {
      idx_out[q] = hi[q];
      if (best_out) best_out[q] = hb[q];
      if (second_out) second_out[q] = hsd[q];
    }
    *last_pivot = cnt > 0 ? hb[cnt - 1] : 0.0;
    *truncated = cnt < b ? 1 : 0;
  });
}

int itercur_select_device(const double* dM, int64_t rows, int64_t cols, int64_t ldm, int64_t b, int32_t is_columns,
                          double pivot_floor, const int64_t* exclude, int64_t n_exclude, int64_t* idx_out,
                          int64_t* n_idx, int32_t* truncated, double* last_pivot, double* best_out,
                          double* second_out, void* stream) {
  return select_impl(dM, rows, cols, ldm, b, is_columns, pivot_floor, exclude, n_exclude, idx_out, n_idx, truncated,
                     last_pivot, best_out, second_out, stream, ITERCUR_PIVOT_LUPP);
}

int itercur_select_qrcp_device(const double* dM, int64_t rows, int64_t cols, int64_t ldm, int64_t b,
                               int32_t is_columns, double pivot_floor, const int64_t* exclude, int64_t n_exclude,
                               int64_t* idx_out, int64_t* n_idx, int32_t* truncated, double* last_pivot,
                               double* best_out, double* second_out, void* stream) {
  return select_impl(dM, rows, cols, ldm, b, is_columns, pivot_floor, exclude, n_exclude, idx_out, n_idx, truncated,
                     last_pivot, best_out, second_out, stream, ITERCUR_PIVOT_QRCP);
}

int itercur_time_sketch_kernel(const double* dA, int64_t m, int64_t n, int64_t lda, int64_t b, int32_t kind,
                               int32_t reps, void* stream, double* ms_per_launch, int32_t* ctas, int32_t* splits,
                               int32_t* uses_tma) {
  return guarded([&] {
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    configure_mempool_once();
    g_alloc_stream = st;
    const int64_t c = sketch_rows(b), cp = round_up(c, 8), ldg = round_up(m, 32);
    const int k = kind == ITERCUR_SKETCH_SPARSE_SIGN ? kSketchSparseSign : kSketchGaussian;
    DevBuf<double> S, Y, wsb, scal;
    Y.alloc(static_cast<size_t>(cp) * n);
    scal.alloc(2);
    SketchLaunchInfo info;
    const int smode = sparse_sketch_mode(k, c, cp, zeta_effective(k, 8, c), dA, lda);
    const bool sparse = smode == kSparseList;
    SketchBuffers sb;
    if (smode == kSparseUmma) {
      wsb.alloc(sparse_sketch_umma_workspace_elems(m, n, cp));
      CK(run_sketch_apply_sparse_umma(dA, m, n, lda, 0, c, cp, zeta_effective(k, 8, c), 1.0, Y.p, wsb.p,
                                      static_cast<int64_t>(wsb.count), SketchStats{scal.p, scal.p + 1}, st, &info,
                                      false, false));
    } else if (smode == kSparseImma) {
      wsb.alloc(sparse_sketch_imma_workspace_elems(m, n, cp));
      CK(run_sketch_apply_sparse_imma(dA, m, n, lda, 0, c, cp, zeta_effective(k, 8, c), 1.0, Y.p, wsb.p,
                                      static_cast<int64_t>(wsb.count), SketchStats{scal.p, scal.p + 1}, st, &info,
                                      false, false));
    } else if (!sparse) {
      S.alloc(static_cast<size_t>(cp) * ldg);
      const int64_t wse = sketch_workspace_elems(m, n, cp);
      wsb.alloc(wse);
      CK(launch_gen_sketch_operator(S.p, cp, ldg, c, m, 0, k, 8, st));
    }
    // the sparse path is timed whole (operator lists + apply + norm reductions); the dense
    // path times its DMMA kernel alone
    auto once = [&]() {
      if (smode == kSparseUmma)
        CK(run_sketch_apply_sparse_umma(dA, m, n, lda, 0, c, cp, zeta_effective(k, 8, c), 1.0, Y.p, wsb.p,
                                        static_cast<int64_t>(wsb.count), SketchStats{scal.p, scal.p + 1}, st, &info,
                                        true, true));
      else if (smode == kSparseImma)  // the integer-path kernel alone (operator already generated)
        CK(run_sketch_apply_sparse_imma(dA, m, n, lda, 0, c, cp, zeta_effective(k, 8, c), 1.0, Y.p, wsb.p,
                                        static_cast<int64_t>(wsb.count), SketchStats{scal.p, scal.p + 1}, st, &info,
                                        true, true));
      else if (sparse)
        apply_sketch(dA, m, n, lda, k, 8, 0, kStreamSketch, c, cp, Y.p, SketchStats{scal.p, scal.p + 1}, sb, st, &info);
      else
        CK(run_sketch_dmma_only(dA, m, n, lda, S.p, ldg, cp, Y.p, wsb.p, static_cast<int64_t>(wsb.count), st, &info));
    };
    once();  // warm-up
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    for (int q = 0; q < reps; ++q) once();
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_per_launch = ms / std::max(reps, 1);
    if (ctas) *ctas = info.ctas;
    if (splits) *splits = info.splits;
    if (uses_tma) *uses_tma = info.tma ? 1 : 0;
  });
}

int itercur_time_lupp(int64_t rows, int32_t steps, int32_t reps, int32_t force_path, void* stream,
                      double* us_per_launch, int32_t* path_used) {
  return guarded([&] {
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    configure_mempool_once();
    g_alloc_stream = st;
    if (rows < 1 || steps < 1) fail(ITERCUR_E_INVALID_ARGUMENT, "rows and steps must be positive");
    const int64_t ldw = even(rows);
    DevBuf<double> W0, W;
    W0.alloc(static_cast<size_t>(ldw) * steps);
    W.alloc(static_cast<size_t>(ldw) * steps);
    CK(launch_gaussian_matrix(ldw, steps, 12345, 3, W0.p, st));
    DevBuf<uint8_t> mask;
    mask.alloc(rows);
    CK(cudaMemsetAsync(mask.p, 0, rows, st));
    DevBuf<char> scratch, outs;
    scratch.alloc(lupp_scratch_bytes(steps));
    CK(lupp_scratch_init(scratch.p, st));
    outs.alloc(sizeof(int64_t) * steps * 3 + 16);
    LuppArgs la{};
    la.W = W.p;
    la.rows = rows;
    la.ldw = ldw;
    la.cols_max = steps;
    la.mask = mask.p;
    la.epoch = 2;
    la.d_norm_sq = nullptr;
    la.pivot_floor = 1e-13;
    la.d_idx = reinterpret_cast<int64_t*>(outs.p);
    la.d_best = reinterpret_cast<double*>(la.d_idx + steps);
    la.d_second = la.d_best + steps;
    la.d_count = reinterpret_cast<int*>(la.d_second + steps);
    set_lupp_force_path(force_path);
    int used = 0;
    CK(cudaMemcpyAsync(W.p, W0.p, sizeof(double) * ldw * steps, cudaMemcpyDeviceToDevice, st));
    CK(run_lupp_with_scratch(la, scratch.p, st, &used));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float total = 0.f;
    for (int q = 0; q < reps; ++q) {
      CK(cudaMemcpyAsync(W.p, W0.p, sizeof(double) * ldw * steps, cudaMemcpyDeviceToDevice, st));
      CK(cudaEventRecord(e0, st));
      CK(run_lupp_with_scratch(la, scratch.p, st, &used));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      total += ms;
    }
    set_lupp_force_path(0);
    // one traced launch: per-step phase cycles of CTA 0 (the cluster kernel records them only
    // in an instrumented build: ITERCUR_NVCC_EXTRA=-DITERCUR_LUPP_INSTRUMENT)
    if (env_flag("ITERCUR_LUPP_TRACE")) {
      DevBuf<long long> tr;
      tr.alloc(static_cast<size_t>(steps) * 16);
      CK(cudaMemsetAsync(tr.p, 0, sizeof(long long) * steps * 16, st));
      set_lupp_force_path(force_path);
      set_lupp_debug_trace(tr.p);
      CK(cudaMemcpyAsync(W.p, W0.p, sizeof(double) * ldw * steps, cudaMemcpyDeviceToDevice, st));
      CK(run_lupp_with_scratch(la, scratch.p, st, &used));
      set_lupp_debug_trace(nullptr);
      set_lupp_force_path(0);
      std::vector<long long> h(static_cast<size_t>(steps) * 16);
      CK(cudaMemcpyAsync(h.data(), tr.p, sizeof(long long) * steps * 16, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (used <= -300000) {  // resident kernel, per step s (thread 0 unless noted): [0] after B1, [1] after B2,
        // [2] CTA argmax, [3] record row stored, [4] lane 1 reciprocal stored, [5] published, [6] headers, [7] tail
        for (int q = 0; q + 1 < steps; ++q) {
          const long long* v = h.data() + q * 8;
          const long long* w = v + 8;
          fprintf(stderr,
                  "lupp resident step %d: B1->B2 %lld argmax %lld row %lld (rcp %lld) pub-end %lld headers %lld tail %lld "
                  "->B1 %lld | step %lld\n",
                  q, v[1] - v[0], v[2] - v[1], v[3] - v[2], v[4] - v[2], v[5] - v[3], w[6] - v[5], w[7] - w[6],
                  w[0] - w[7], w[0] - v[0]);
        }
      } else if (used <= -200000) {  // panel kernel (8 slots per step)
        for (int q = 0; q + 1 < steps; ++q) {
          const long long* v = h.data() + q * 8;
          fprintf(stderr,
                  "lupp panel step %d: reduce %lld pivot-row %lld rows %lld panel-end %lld cand %lld barrier %lld "
                  "step %lld\n",
                  q, v[1] - v[0], v[2] - v[1], v[3] - v[2], v[4] - v[3], v[5] - v[4], v[8] - v[5], v[8] - v[0]);
        }
      } else if (used <= -100) {  // cluster v2 layout (16 slots per step)
        for (int q = 0; q + 1 < steps; ++q) {
          const long long* v = h.data() + q * 16;
          fprintf(stderr,
                  "lupp v2 step %d: [t32] eager %lld wcand %lld | [t0] B1-released %lld read-wc %lld argmax %lld vals "
                  "%lld st.async %lld wait %lld read-in %lld argmax %lld tail %lld | B2-released(t32) %lld | step %lld [probe %lld]\n",
                  q, v[1] - v[0], v[2] - v[1], v[3] - v[2], v[10] - v[3], v[11] - v[10], v[12] - v[11], v[4] - v[12],
                  v[5] - v[4], v[13] - v[5], v[14] - v[13], v[15] - v[14], v[8] - v[15], v[16] - v[0], v[9] / 100);
        }
      } else
      for (int q = 0; q + 1 < steps; ++q) {
        const long long* v = h.data() + q * 8;
        fprintf(stderr,
                "lupp trace step %d: col1 %lld wcand %lld B2 %lld publish %lld exchange %lld deferred %lld "
                "B1(after exch) %lld step %lld\n",
                q, v[1] - v[0], v[2] - v[1], v[3] - v[2], v[4] - v[3], v[5] - v[4], v[6] - v[2], v[7] - v[5],
                v[8] - v[0]);
      }
    }
    if (env_flag("ITERCUR_LUPP_GTRACE")) {  // resident path: skew of the per-step exchange over the CTAs
      const int G = kNumSMs;
      DevBuf<long long> tr;
      tr.alloc(static_cast<size_t>(steps) * G * 4);
      CK(cudaMemsetAsync(tr.p, 0, sizeof(long long) * steps * G * 4, st));
      set_lupp_force_path(force_path);
      set_lupp_grid_trace(tr.p);
      CK(cudaMemcpyAsync(W.p, W0.p, sizeof(double) * ldw * steps, cudaMemcpyDeviceToDevice, st));
      CK(run_lupp_with_scratch(la, scratch.p, st, &used));
      set_lupp_grid_trace(nullptr);
      set_lupp_force_path(0);
      std::vector<long long> h(static_cast<size_t>(steps) * G * 4);
      CK(cudaMemcpyAsync(h.data(), tr.p, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      const int Gu = used <= -300000 ? -used - 300000 : G;
      for (int q = 1; q + 1 < steps; ++q) {
        long long pmin = LLONG_MAX, pmax = 0, hmin = LLONG_MAX, hmax = 0, tmin = LLONG_MAX, tmax = 0, last = 0;
        long long cmax = 0, csum = 0;
        for (int g = 0; g < Gu; ++g) {
          const long long* v = h.data() + (static_cast<size_t>(q) * G + g) * 4;
          const long long* pv = h.data() + (static_cast<size_t>(q - 1) * G + g) * 4;
          if (v[0] > pmax) pmax = v[0], last = g;
          pmin = std::min(pmin, v[0]);
          hmin = std::min(hmin, v[1]);
          hmax = std::max(hmax, v[1]);
          tmin = std::min(tmin, v[2]);
          tmax = std::max(tmax, v[2]);
          const long long c = v[0] - pv[2];  // this CTA: tail of step q-1 seen -> record q published
          cmax = std::max(cmax, c);
          csum += c;
        }
        fprintf(stderr,
                "gtrace step %d: publish spread %lld ns (last CTA %lld) | last publish -> headers seen %lld..%lld ns | "
                "headers -> tail %lld..%lld ns | tail seen -> publish mean %lld max %lld ns\n",
                q, pmax - pmin, last, hmin - pmax, hmax - pmax, tmin - hmin, tmax - hmax, csum / Gu, cmax);
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *us_per_launch = 1e3 * total / std::max(reps, 1);
    if (path_used) *path_used = used;
  });
}

int itercur_csr_to_dense_device(int64_t rows, int64_t cols, const int64_t* dRowPtr, const int64_t* dColIdx,
                                const double* dValues, double* dOut, int64_t ld, void* stream) {
  return guarded([&] {
    require_device();
    if (rows < 0 || cols < 0 || ld < std::max<int64_t>(rows, 1))
      fail(ITERCUR_E_INVALID_ARGUMENT, "csr_to_dense: invalid shape or leading dimension");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CK(cudaMemsetAsync(dOut, 0, sizeof(double) * ld * cols, st));
    CK(launch_csr_to_dense(rows, dRowPtr, dColIdx, dValues, dOut, ld, st));
  });
}

int itercur_lupp_dist_step(double* dW, int64_t rows, int64_t ldw, int32_t steps, int32_t s, const double* dPivotRow,
                           int64_t pivot_local_row, uint8_t* dLive, int64_t row_offset, double* dCand, void* stream) {
  return guarded([&] {
    require_device();
    if (rows < 0 || steps < 1 || s < 0 || s >= steps || ldw < std::max<int64_t>(rows, 1) || (s > 0 && !dPivotRow))
      fail(ITERCUR_E_INVALID_ARGUMENT, "lupp_dist_step: invalid arguments");
    CK(launch_lupp_dist_step(dW, rows, ldw, steps, s, s > 0 ? dPivotRow : nullptr, pivot_local_row, dLive, row_offset,
                             dCand, static_cast<cudaStream_t>(stream)));
  });
}

int itercur_gemm_device(int64_t M, int64_t N, int64_t K, const double* dA, int64_t lda, const double* dB, int64_t ldb,
                        const double* dBase, int64_t ldbase, double alpha, double* dC, int64_t ldc, void* stream) {
  return guarded([&] {
    require_device();
    if (M < 0 || N < 0 || K < 0 || (lda & 1) || (reinterpret_cast<uintptr_t>(dA) & 15) || ldc < std::max<int64_t>(M, 1) ||
        ldb < std::max<int64_t>(K, 1) || (dBase && ldbase < std::max<int64_t>(M, 1)) || N > (1 << 30))
      fail(ITERCUR_E_INVALID_ARGUMENT, "gemm_device: invalid shape, leading dimension or alignment");
    if (M == 0 || N == 0) return;
    TsGemmParams p;
    p.M = M;
    p.K = K;
    p.N = static_cast<int>(N);
    p.A = dA;
    p.lda = lda;
    p.B = dB;
    p.bsk = 1;
    p.bsn = ldb;
    p.base_mode = dBase ? kBaseContigCols : kBaseNone;
    p.src = dBase;
    p.lds = ldbase;
    p.col0 = 0;
    p.alpha = alpha;
    p.out_mode = kOutColMajor;
    p.C0 = dC;
    p.ldc0 = ldc;
    CK(run_ts_gemm(p, static_cast<cudaStream_t>(stream)));
  });
}

int itercur_block_lu_device(double* dD, int64_t w, int64_t ldd, void* stream) {
  return guarded([&] {
    require_device();
    if (w < 0 || w > 4096 || ldd < std::max<int64_t>(w, 1)) fail(ITERCUR_E_INVALID_ARGUMENT, "block_lu: invalid shape");
    CK(launch_dense_lu(dD, static_cast<int>(w), ldd, static_cast<cudaStream_t>(stream)));
  });
}

int itercur_rows_lu_solve_device(const double* dX, int64_t ldx, int64_t M, const double* dLU, int64_t ldd, int64_t w,
                                 double* dOut, int64_t ldo, void* stream) {
  return guarded([&] {
    require_device();
    if (M < 0 || w < 0 || w > 4096 || ldx < std::max<int64_t>(M, 1) || ldo < std::max<int64_t>(M, 1) ||
        ldd < std::max<int64_t>(w, 1))
      fail(ITERCUR_E_INVALID_ARGUMENT, "rows_lu_solve: invalid shape");
    CK(launch_rows_lu_solve(dX, ldx, M, dLU, ldd, nullptr, static_cast<int>(w), dOut, ldo,
                            static_cast<cudaStream_t>(stream), nullptr, 0));
  });
}

int itercur_time_gemm(int64_t M, int32_t N, int64_t K, int32_t reps, void* stream, double* us_per_launch) {
  return guarded([&] {
    require_device();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    configure_mempool_once();
    g_alloc_stream = st;
    const int64_t ldl = even(M);
    DevBuf<double> Lm, Bm, Cm, Asrc;
    DevBuf<int64_t> idx;
    Lm.alloc(static_cast<size_t>(ldl) * std::max<int64_t>(K, 1));
    Bm.alloc(static_cast<size_t>(std::max<int64_t>(K, 1)) * N);
    Cm.alloc(static_cast<size_t>(ldl) * N);
    Asrc.alloc(static_cast<size_t>(ldl) * N);
    idx.alloc(N);
    CK(launch_gaussian_matrix(ldl, std::max<int64_t>(K, 1), 1, 3, Lm.p, st));
    CK(launch_gaussian_matrix(std::max<int64_t>(K, 1), N, 2, 3, Bm.p, st));
    CK(launch_gaussian_matrix(ldl, N, 3, 3, Asrc.p, st));
    std::vector<int64_t> h(N);
    for (int q = 0; q < N; ++q) h[q] = q;
    CK(cudaMemcpyAsync(idx.p, h.data(), sizeof(int64_t) * N, cudaMemcpyHostToDevice, st));
    TsGemmParams p;
    p.M = M;
    p.K = K;
    p.N = N;
    p.A = Lm.p;
    p.lda = ldl;
    p.B = Bm.p;
    p.bsk = 1;
    p.bsn = std::max<int64_t>(K, 1);
    p.base_mode = kBaseGatherCols;
    p.src = Asrc.p;
    p.lds = ldl;
    p.idx = idx.p;
    p.alpha = -1.0;
    p.out_mode = kOutColMajor;
    p.C0 = Cm.p;
    p.ldc0 = ldl;
    CK(run_ts_gemm(p, st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    for (int q = 0; q < reps; ++q) CK(run_ts_gemm(p, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *us_per_launch = 1e3 * ms / std::max(reps, 1);
  });
}

}  // extern "C"

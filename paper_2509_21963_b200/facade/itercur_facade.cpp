// itercur_facade.cpp — the C++ API of include/itercur/driver_b200.hpp over the engine's C-ABI
// (include/itercur_b200.h). Type and exception mapping only: every computation runs in
// libitercur_b200.so on the B200. Built by paper_2509_21963_b200/build.py into
// libitercur_facade.so (g++, links libitercur_b200.so with an $ORIGIN rpath).
#include "itercur/driver_b200.hpp"

#include <algorithm>
#include <cmath>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>

#include "itercur_b200.h"

#define ITERCUR_FACADE_API __attribute__((visibility("default")))

namespace itercur {
namespace detail {

// The engine's exception classes, with its messages (the reference's texts).
[[noreturn]] void rethrow(int code) {
  const std::string msg = itercur_last_error();
  switch (code) {
    case ITERCUR_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ITERCUR_E_OUT_OF_RANGE: throw std::out_of_range(msg);
    case ITERCUR_E_DOMAIN: throw std::domain_error(msg);
    case ITERCUR_E_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}
void check(int code) {
  if (code != ITERCUR_OK) rethrow(code);
}

// Owns one engine run (CurFactors + RunTrace + device factors); freed with the last reference.
struct RunRef {
  itercur_run* run = nullptr;
  explicit RunRef(itercur_run* r) : run(r) {}
  RunRef(const RunRef&) = delete;
  RunRef& operator=(const RunRef&) = delete;
  ~RunRef() {
    if (run) itercur_run_free(run);
  }
};

enum class Kind { HostDense, Csr, Device, RunC, RunR };

struct Payload {
  Kind kind = Kind::HostDense;
  Index rows = 0, cols = 0;
  DenseMatrix dense;  // HostDense
  CsrData csr;        // Csr
  const double* d = nullptr;  // Device
  Index ld = 0;
  std::shared_ptr<const RunRef> run;  // RunC / RunR: gathered from the run's A on first use
  mutable std::once_flag once;
  mutable DenseMatrix cache;
};

const DenseMatrix& host_dense(const Payload& p) {
  if (p.kind == Kind::HostDense) return p.dense;
  std::call_once(p.once, [&] {
    DenseMatrix out(p.rows, p.cols);
    switch (p.kind) {
      case Kind::Csr:  // CsrData::to_dense (matrix.cpp:113-131)
        for (Index i = 0; i < p.rows; ++i)
          for (Index q = p.csr.row_ptr[static_cast<size_t>(i)]; q < p.csr.row_ptr[static_cast<size_t>(i) + 1]; ++q)
            out(i, p.csr.col_idx[static_cast<size_t>(q)]) = p.csr.values[static_cast<size_t>(q)];
        break;
      case Kind::Device:
        if (p.ld == p.rows) {
          check(itercur_copy_to_host(out.data(), p.d, sizeof(double) * p.rows * p.cols));
        } else {
          for (Index j = 0; j < p.cols; ++j)
            check(itercur_copy_to_host(out.data() + j * p.rows, p.d + j * p.ld, sizeof(double) * p.rows));
        }
        break;
      case Kind::RunC:
        if (out.size()) check(itercur_run_c_matrix(p.run->run, out.data()));
        break;
      case Kind::RunR:
        if (out.size()) check(itercur_run_r_matrix(p.run->run, out.data()));
        break;
      default:
        break;
    }
    p.cache = std::move(out);
  });
  return p.cache;
}

int32_t pivot_kind(const SelectionMethod& m) {
  switch (m.kind) {
    case PivotKind::Lupp: return ITERCUR_PIVOT_LUPP;
    case PivotKind::Qrcp: return ITERCUR_PIVOT_QRCP;
    case PivotKind::Osinsky: return ITERCUR_PIVOT_OSINSKY;
  }
  return ITERCUR_PIVOT_LUPP;
}

IterationRecord to_record(const itercur_iteration_record& x) {
  IterationRecord rec;
  rec.k = x.k;
  rec.rho = x.rho;
  rec.cols_added = x.cols_added;
  rec.rows_added = x.rows_added;
  rec.col_truncated = x.col_truncated != 0;
  rec.row_truncated = x.row_truncated != 0;
  rec.select_cols_s = x.select_cols_s;
  rec.row_residual_s = x.row_residual_s;
  rec.select_rows_s = x.select_rows_s;
  rec.core_s = x.core_s;
  rec.downdate_s = x.downdate_s;
  return rec;
}

void run_indices(const itercur_run* run, IndexList& I, IndexList& J) {
  const Index r = itercur_run_rank(run);
  I.assign(static_cast<size_t>(r), 0);
  J.assign(static_cast<size_t>(r), 0);
  check(itercur_run_indices(run, I.data(), J.data()));
}

MatrixHandle run_matrix(std::shared_ptr<const RunRef> ref, Kind kind, Index rows, Index cols) {
  auto p = std::make_shared<Payload>();
  p->kind = kind;
  p->rows = rows;
  p->cols = cols;
  p->run = std::move(ref);
  return MatrixHandle(std::shared_ptr<const Payload>(std::move(p)));
}

MatrixHandle host_matrix(DenseMatrix d) {
  auto p = std::make_shared<Payload>();
  p->kind = Kind::HostDense;
  p->rows = d.rows();
  p->cols = d.cols();
  p->dense = std::move(d);
  return MatrixHandle(std::shared_ptr<const Payload>(std::move(p)));
}

// Runs the engine on A with the given config (device entry for device handles, host entry
// otherwise; CSR densifies as the reference's to_dense would).
itercur_run* run_engine(const MatrixHandle& A, itercur_config& c) {
  const Payload& p = *A.payload();
  itercur_run* run = nullptr;
  int rc;
  if (p.kind == Kind::Device) {
    rc = itercur_iterative_cur_device(p.d, p.rows, p.cols, p.ld, &c, nullptr, &run);
  } else {
    const DenseMatrix& d = host_dense(p);
    rc = itercur_iterative_cur_host(d.data(), p.rows, p.cols, std::max<Index>(p.rows, 1), &c, &run);
  }
  if (rc != ITERCUR_OK) rethrow(rc);
  return run;
}

CurFactors factors_of(const std::shared_ptr<const RunRef>& ref) {
  CurFactors f;
  run_indices(ref->run, f.row_indices, f.col_indices);
  const Index r = f.rank(), m = itercur_run_rows(ref->run), n = itercur_run_cols(ref->run);
  f.C = run_matrix(ref, Kind::RunC, m, r);
  f.R = run_matrix(ref, Kind::RunR, r, n);
  f.core = FactoredPinv(ref, r);
  return f;
}

// IterationObserver bridge: an eager snapshot of the factors after the iteration (the run goes on
// after the callback, so nothing here may refer back to it lazily).
struct ObserverCtx {
  const IterationObserver* fn = nullptr;
  std::exception_ptr error;
};
int observer_trampoline(void* user, const itercur_run* run, const itercur_iteration_record* rec) {
  auto* ctx = static_cast<ObserverCtx*>(user);
  try {
    CurFactors f;
    run_indices(run, f.row_indices, f.col_indices);
    const Index r = f.rank(), m = itercur_run_rows(run), n = itercur_run_cols(run);
    DenseMatrix c(m, r), rr(r, n), core(r, r);
    if (r) {
      check(itercur_run_c_matrix(run, c.data()));
      check(itercur_run_r_matrix(run, rr.data()));
      check(itercur_run_core_matrix(run, core.data()));
    }
    f.C = host_matrix(std::move(c));
    f.R = host_matrix(std::move(rr));
    f.core = FactoredPinv(std::move(core));
    (*ctx->fn)(f, to_record(*rec));
    return 0;
  } catch (...) {
    ctx->error = std::current_exception();
    return 1;
  }
}

}  // namespace detail

using detail::check;
using detail::Kind;
using detail::Payload;

// ------------------------------------------------------------------ MatrixHandle
ITERCUR_FACADE_API MatrixHandle::MatrixHandle() : p_(std::make_shared<Payload>()) {}

ITERCUR_FACADE_API MatrixHandle::MatrixHandle(DenseMatrix dense) {
  for (Index q = 0; q < dense.size(); ++q)
    if (!std::isfinite(dense.data()[q])) throw std::invalid_argument("matrix contains non-finite entries");
  p_ = detail::host_matrix(std::move(dense)).payload();
}

ITERCUR_FACADE_API MatrixHandle::MatrixHandle(Index rows, Index cols, std::vector<Index> row_ptr,
                                              std::vector<Index> col_idx, std::vector<double> values) {
  // matrix.cpp:79-104
  if (rows < 0 || cols < 0) throw std::invalid_argument("negative matrix dimension");
  if (static_cast<Index>(row_ptr.size()) != rows + 1) throw std::invalid_argument("row_ptr must have rows+1 entries");
  if (row_ptr.front() != 0 || row_ptr.back() != static_cast<Index>(values.size()))
    throw std::invalid_argument("row_ptr must start at 0 and end at nnz");
  if (col_idx.size() != values.size()) throw std::invalid_argument("col_idx and values must have equal length");
  for (Index i = 0; i < rows; ++i) {
    if (row_ptr[static_cast<size_t>(i) + 1] < row_ptr[static_cast<size_t>(i)])
      throw std::invalid_argument("row_ptr must be nondecreasing");
    for (Index q = row_ptr[static_cast<size_t>(i)]; q < row_ptr[static_cast<size_t>(i) + 1]; ++q) {
      const Index j = col_idx[static_cast<size_t>(q)];
      if (j < 0 || j >= cols)
        throw std::out_of_range("csr column index " + std::to_string(j) + " out of range [0, " + std::to_string(cols) + ")");
      if (q > row_ptr[static_cast<size_t>(i)] && j <= col_idx[static_cast<size_t>(q) - 1])
        throw std::invalid_argument("csr column indices must be strictly increasing within each row");
    }
  }
  for (double v : values)
    if (!std::isfinite(v)) throw std::invalid_argument("matrix contains non-finite entries");
  auto p = std::make_shared<Payload>();
  p->kind = Kind::Csr;
  p->rows = rows;
  p->cols = cols;
  p->csr = CsrData{rows, cols, std::move(row_ptr), std::move(col_idx), std::move(values)};
  p_ = std::move(p);
}

ITERCUR_FACADE_API MatrixHandle MatrixHandle::device(const double* d_data, Index rows, Index cols, Index ld) {
  if (rows < 0 || cols < 0 || ld < std::max<Index>(rows, 1)) throw std::invalid_argument("invalid device matrix shape");
  auto p = std::make_shared<Payload>();
  p->kind = Kind::Device;
  p->rows = rows;
  p->cols = cols;
  p->d = d_data;
  p->ld = ld;
  return MatrixHandle(std::shared_ptr<const Payload>(std::move(p)));
}

ITERCUR_FACADE_API Index MatrixHandle::rows() const { return p_->rows; }
ITERCUR_FACADE_API Index MatrixHandle::cols() const { return p_->cols; }
ITERCUR_FACADE_API bool MatrixHandle::is_sparse() const { return p_->kind == Kind::Csr; }
ITERCUR_FACADE_API bool MatrixHandle::is_device() const { return p_->kind == Kind::Device; }
ITERCUR_FACADE_API Index MatrixHandle::nnz() const {
  return p_->kind == Kind::Csr ? static_cast<Index>(p_->csr.values.size()) : p_->rows * p_->cols;
}
ITERCUR_FACADE_API const DenseMatrix& MatrixHandle::dense_data() const {
  if (p_->kind == Kind::Csr) throw std::logic_error("dense_data() on a sparse matrix");
  return detail::host_dense(*p_);
}
ITERCUR_FACADE_API const CsrData& MatrixHandle::csr_data() const {
  if (p_->kind != Kind::Csr) throw std::logic_error("csr_data() on a dense matrix");
  return p_->csr;
}
ITERCUR_FACADE_API DenseMatrix MatrixHandle::to_dense() const { return detail::host_dense(*p_); }

ITERCUR_FACADE_API double fro_norm(const MatrixHandle& A) {
  const Payload& p = *A.payload();
  if (p.kind == Kind::Device) {
    double out = 0.0;
    check(itercur_fro_norm_device(p.d, p.rows, p.cols, p.ld, nullptr, &out));
    return out;
  }
  double out = 0.0;
  if (p.kind == Kind::Csr) {  // ||values||: the stored entries as one column
    const Index nnz = static_cast<Index>(p.csr.values.size());
    if (nnz) check(itercur_fro_norm_host(p.csr.values.data(), nnz, 1, nnz, &out));
    return out;
  }
  const DenseMatrix& d = detail::host_dense(p);
  check(itercur_fro_norm_host(d.data(), d.rows(), d.cols(), std::max<Index>(d.rows(), 1), &out));
  return out;
}

// ------------------------------------------------------------------ FactoredPinv
ITERCUR_FACADE_API FactoredPinv::FactoredPinv(DenseMatrix inverse)
    : host_(std::make_shared<const DenseMatrix>(std::move(inverse))), r_(host_->rows()) {}

namespace {
DenseMatrix apply(const std::shared_ptr<const detail::RunRef>& run, const std::shared_ptr<const DenseMatrix>& host,
                  Index r, const DenseMatrix& rhs, bool transposed) {
  if (rhs.rows() != r)
    throw std::invalid_argument(std::string(transposed ? "apply_pinv_right: expected " : "apply_pinv_left: expected ") +
                                std::to_string(r) + (transposed ? " columns, got " : " rows, got ") +
                                std::to_string(rhs.rows()));
  if (!run && !host) throw std::logic_error("FactoredPinv is empty");
  DenseMatrix out(r, rhs.cols());
  if (r == 0 || rhs.cols() == 0) return out;
  if (run) {
    check(itercur_run_core_apply(run->run, transposed ? 1 : 0, rhs.data(), rhs.cols(), r, out.data(), r));
    return out;
  }
  // observer snapshot: the materialised inverse (copied out of the engine during the callback),
  // applied on the device
  check(itercur_dense_apply_host(host->data(), r, transposed ? 1 : 0, rhs.data(), rhs.cols(), out.data()));
  return out;
}
}  // namespace

ITERCUR_FACADE_API DenseMatrix FactoredPinv::solve(const DenseMatrix& rhs) const {
  return apply(run_, host_, r_, rhs, false);
}
ITERCUR_FACADE_API DenseMatrix FactoredPinv::solve_transposed(const DenseMatrix& rhs) const {
  return apply(run_, host_, r_, rhs, true);
}
ITERCUR_FACADE_API DenseMatrix FactoredPinv::materialize() const {
  if (host_) return *host_;
  if (!run_) throw std::logic_error("FactoredPinv is empty");
  DenseMatrix out(r_, r_);
  if (r_) check(itercur_run_core_matrix(run_->run, out.data()));
  return out;
}

// ------------------------------------------------------------------ driver
ITERCUR_FACADE_API const char* to_string(RunStatus status) {
  switch (status) {
    case RunStatus::Converged: return "Converged";
    case RunStatus::MaxRank: return "MaxRank";
    case RunStatus::ResidualExhausted: return "ResidualExhausted";
  }
  return "Unknown";
}

ITERCUR_FACADE_API double adjusted_threshold(double epsilon, double delta, double alpha, Index c) {
  double out = 0.0;
  check(itercur_adjusted_threshold(epsilon, delta, alpha, c, &out));
  return out;
}

ITERCUR_FACADE_API double gratton_tail(Index c, double tau) {
  double out = 0.0;
  check(itercur_gratton_tail(c, tau, &out));
  return out;
}

ITERCUR_FACADE_API CurResult iterative_cur(const MatrixHandle& A, const StoppingConfig& cfg,
                                           const SelectionMethod& col_method, const SelectionMethod& row_method,
                                           std::uint64_t seed, const IterationObserver& observer) {
  itercur_config c;
  itercur_config_default(&c);
  c.epsilon = cfg.epsilon;
  c.b = cfg.b;
  c.delta = cfg.delta;
  c.alpha = cfg.alpha;
  c.risk_adjust = cfg.risk_adjust ? 1 : 0;
  c.max_rank = cfg.max_rank;
  c.max_iters = cfg.max_iters;
  c.col_method = detail::pivot_kind(col_method);
  c.row_method = detail::pivot_kind(row_method);
  c.pivot_floor = col_method.pivot_floor;
  c.row_pivot_floor = row_method.pivot_floor;
  c.seed = seed;
  c.sketch_kind = cfg.sketch == SketchKind::SparseSign ? ITERCUR_SKETCH_SPARSE_SIGN : ITERCUR_SKETCH_GAUSSIAN;
  c.sparse_nnz = cfg.sparse_nnz;
  detail::ObserverCtx ctx;
  if (observer) {
    ctx.fn = &observer;
    c.observer = &detail::observer_trampoline;
    c.observer_user = &ctx;
  }
  itercur_run* raw = nullptr;
  try {
    raw = detail::run_engine(A, c);
  } catch (...) {
    if (ctx.error) std::rethrow_exception(ctx.error);  // the observer's own exception, as the reference propagates it
    throw;
  }
  auto ref = std::make_shared<const detail::RunRef>(raw);
  CurResult out;
  out.factors = detail::factors_of(ref);
  RunTrace& t = out.trace;
  t.status = static_cast<RunStatus>(itercur_run_status(raw));
  t.final_rho = itercur_run_final_rho(raw);
  t.threshold = itercur_run_threshold(raw);
  t.sketch_s = itercur_run_sketch_seconds(raw);
  t.total_s = itercur_run_total_seconds(raw);
  t.note = itercur_run_note(raw);
  std::vector<itercur_iteration_record> recs(static_cast<size_t>(itercur_run_num_iterations(raw)));
  if (!recs.empty()) check(itercur_run_iterations(raw, recs.data()));
  for (const auto& x : recs) t.iterations.push_back(detail::to_record(x));
  return out;
}

ITERCUR_FACADE_API double true_relative_error(const MatrixHandle& A, const CurFactors& cur) {
  if (cur.empty()) return fro_norm(A) == 0.0 ? 0.0 : 1.0;  // driver.cpp:170-172
  const auto& ref = cur.core.run_ref();
  if (!ref)
    throw std::logic_error("true_relative_error: the factors of an observer snapshot are host copies; "
                           "evaluate the finished run's factors");
  const Payload& p = *A.payload();
  double out = 0.0;
  if (p.kind == Kind::Device) {
    check(itercur_true_relative_error_matrix(ref->run, p.d, p.rows, p.cols, p.ld, 1, &out));
  } else {
    const DenseMatrix& d = detail::host_dense(p);
    check(itercur_true_relative_error_matrix(ref->run, d.data(), p.rows, p.cols, std::max<Index>(p.rows, 1), 0, &out));
  }
  return out;
}

ITERCUR_FACADE_API CurFactors slupp_cur(const MatrixHandle& A, Index rank, std::uint64_t seed) {
  // baselines.cpp:39-62: one sketch of ceil(1.1 r) rows on stream SluppSketch, r LUPP column
  // pivots, LUPP row pivots on A(:, J), the factors — one engine block with b = r
  if (rank < 0 || rank > std::min(A.rows(), A.cols())) throw std::invalid_argument("rank must lie in [0, min(m, n)]");
  if (rank == 0) return CurFactors{};
  itercur_config c;
  itercur_config_default(&c);
  c.epsilon = 0.0;
  c.b = rank;
  c.max_rank = rank;
  c.max_iters = 1;
  c.seed = seed;
  c.sketch_stream = 2;
  c.sketch_rows = (11 * rank + 9) / 10;
  auto ref = std::make_shared<const detail::RunRef>(detail::run_engine(A, c));
  CurFactors f = detail::factors_of(ref);
  if (f.empty()) throw std::runtime_error("singular cross block");
  return f;
}

}  // namespace itercur

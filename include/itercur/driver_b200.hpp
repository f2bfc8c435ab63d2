// itercur/driver_b200.hpp — C++ facade of the B200 IterativeCUR engine with the reference's API.
//
// The reference's C++ entry point and types (paths relative to /root/reference/proj):
//
//   itercur::iterative_cur(A, StoppingConfig, SelectionMethod col, SelectionMethod row, seed,
//                          IterationObserver)                include/itercur/driver.hpp:79-81
//   StoppingConfig                                           include/itercur/driver.hpp:18-26
//   RunStatus / IterationRecord / RunTrace / CurResult       include/itercur/driver.hpp:28-59
//   IterationObserver                                        include/itercur/driver.hpp:70-72
//   true_relative_error, adjusted_threshold, gratton_tail    include/itercur/driver.hpp:64-85
//   PivotKind / SelectionMethod                              include/itercur/select.hpp:7-15
//   FactoredPinv / CurFactors                                include/itercur/pinv.hpp:16-66
//   MatrixHandle / CsrData                                   include/itercur/matrix.hpp:17-59
//   slupp_cur                                                include/itercur/baselines.hpp (baselines.cpp:39-62)
//
// Same namespace, names, parameter order, field names and defaults. The Eigen-typed members
// (Eigen is not in this image) become itercur::DenseMatrix, a column-major FP64 matrix with the
// Eigen accessors the reference's callers use (rows/cols/operator()/data/outerStride). Extensions:
// StoppingConfig::sketch / sparse_nnz (sparse-sign sketch) and MatrixHandle::device (a device-
// resident input that never round-trips through the host).
//
// Everything computes on the B200 through the C-ABI in include/itercur_b200.h
// (libitercur_b200.so); this facade (libitercur_facade.so) only maps types and exceptions:
// invalid_argument / out_of_range / domain_error / runtime_error / logic_error, with the
// reference's messages. The core is the engine's exact block-LU inverse of A(I, J), applied on
// the device (FactoredPinv::solve); C and R are gathered from A on the device on first use.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace itercur {

using Index = std::int64_t;
using IndexList = std::vector<Index>;

/// Column-major FP64 matrix (stands in for Eigen::MatrixXd).
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(Index rows, Index cols) : rows_(rows), cols_(cols), v_(static_cast<size_t>(rows * cols), 0.0) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  Index outerStride() const { return rows_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(i + j * rows_)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(i + j * rows_)]; }
  static DenseMatrix Identity(Index n) {
    DenseMatrix e(n, n);
    for (Index i = 0; i < n; ++i) e(i, i) = 1.0;
    return e;
  }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<double> v_;
};

/// Compressed-sparse-row storage (matrix.hpp:17-23).
struct CsrData {
  Index rows = 0;
  Index cols = 0;
  std::vector<Index> row_ptr;
  std::vector<Index> col_idx;
  std::vector<double> values;
};

namespace detail {
struct Payload;
struct RunRef;
}  // namespace detail

/// Dense / CSR / device matrix with value semantics; the payload is immutable and shared.
class MatrixHandle {
 public:
  MatrixHandle();
  /// Wrap a dense host matrix. All entries must be finite (matrix.cpp:73-77).
  explicit MatrixHandle(DenseMatrix dense);
  /// CSR from raw arrays, validated as matrix.cpp:79-104 validates it.
  MatrixHandle(Index rows, Index cols, std::vector<Index> row_ptr, std::vector<Index> col_idx,
               std::vector<double> values);
  /// A column-major device matrix (rows x cols, leading dimension ld) on the current device; not
  /// copied — it must outlive every use of the handle and of factors computed from it.
  static MatrixHandle device(const double* d_data, Index rows, Index cols, Index ld);

  Index rows() const;
  Index cols() const;
  bool is_sparse() const;
  bool is_device() const;
  bool empty() const { return rows() == 0 || cols() == 0; }
  Index nnz() const;
  /// Host dense data (device / factor-backed handles are copied to the host on first use).
  const DenseMatrix& dense_data() const;
  const CsrData& csr_data() const;
  DenseMatrix to_dense() const;

  std::shared_ptr<const detail::Payload> payload() const { return p_; }
  explicit MatrixHandle(std::shared_ptr<const detail::Payload> p) : p_(std::move(p)) {}

 private:
  std::shared_ptr<const detail::Payload> p_;
};

double fro_norm(const MatrixHandle& A);

/// The core A(I, J)^+ in factored form (pinv.hpp:16-40). For the engine's nonsingular cross
/// blocks this is the exact inverse, held as the block-LU factors on the device.
class FactoredPinv {
 public:
  FactoredPinv() = default;
  Index rows() const { return r_; }
  Index cols() const { return r_; }
  Index rank() const { return r_; }
  double tolerance() const { return 0.0; }
  bool valid() const { return run_ != nullptr || host_ != nullptr; }
  /// X^+ * rhs.
  DenseMatrix solve(const DenseMatrix& rhs) const;
  /// (X^T)^+ * rhs.
  DenseMatrix solve_transposed(const DenseMatrix& rhs) const;
  /// Explicit X^+ (export only), FactoredPinv::materialize (pinv.cpp:40-43).
  DenseMatrix materialize() const;

  FactoredPinv(std::shared_ptr<const detail::RunRef> run, Index r) : run_(std::move(run)), r_(r) {}
  explicit FactoredPinv(DenseMatrix inverse);
  const std::shared_ptr<const detail::RunRef>& run_ref() const { return run_; }

 private:
  std::shared_ptr<const detail::RunRef> run_;
  std::shared_ptr<const DenseMatrix> host_;  // materialised inverse (observer snapshots)
  Index r_ = 0;
};

/// C = A(:,J), core = A(I,J)^+, R = A(I,:) (pinv.hpp:57-66).
struct CurFactors {
  IndexList row_indices;  // I
  IndexList col_indices;  // J
  MatrixHandle C;
  FactoredPinv core;
  MatrixHandle R;
  bool empty() const { return col_indices.empty(); }
  Index rank() const { return static_cast<Index>(col_indices.size()); }
};

enum class PivotKind { Lupp, Qrcp, Osinsky };

/// select.hpp:12-15: each method carries its own pivot floor.
struct SelectionMethod {
  PivotKind kind = PivotKind::Lupp;
  double pivot_floor = 1e-13;
};

enum class SketchKind { Gaussian, SparseSign };

/// driver.hpp:18-26, plus the sketch kind (the reference hard-wires Gaussian, sketch.cpp:19).
struct StoppingConfig {
  double epsilon = 1e-6;
  Index b = 50;
  double delta = 0.0;
  double alpha = 0.05;
  bool risk_adjust = false;
  Index max_rank = 0;   // 0 -> min(m, n)
  Index max_iters = 0;  // 0 -> ceil(min(m, n) / b) + 1
  SketchKind sketch = SketchKind::Gaussian;
  int sparse_nnz = 8;
};

enum class RunStatus { Converged, MaxRank, ResidualExhausted };
const char* to_string(RunStatus status);

struct IterationRecord {
  Index k = 0;
  double rho = 1.0;
  Index cols_added = 0;
  Index rows_added = 0;
  bool col_truncated = false;
  bool row_truncated = false;
  double select_cols_s = 0.0;
  double row_residual_s = 0.0;
  double select_rows_s = 0.0;
  double core_s = 0.0;
  double downdate_s = 0.0;
};

struct RunTrace {
  std::vector<IterationRecord> iterations;
  RunStatus status = RunStatus::Converged;
  double final_rho = 1.0;
  double threshold = 0.0;
  double sketch_s = 0.0;
  double total_s = 0.0;
  std::string note;
};

struct CurResult {
  CurFactors factors;
  RunTrace trace;
};

double adjusted_threshold(double epsilon, double delta, double alpha, Index c);
double gratton_tail(Index c, double tau);

/// Invoked with the factors as they stand after each completed iteration (driver.cpp:154).
using IterationObserver = std::function<void(const CurFactors&, const IterationRecord&)>;

CurResult iterative_cur(const MatrixHandle& A, const StoppingConfig& cfg, const SelectionMethod& col_method,
                        const SelectionMethod& row_method, std::uint64_t seed, const IterationObserver& observer = {});

/// ||A - C core R||_F / ||A||_F for the given A (driver.cpp:169-190), on the device.
double true_relative_error(const MatrixHandle& A, const CurFactors& cur);

/// One-shot s-LUPP CUR baseline (baselines.cpp:39-62).
CurFactors slupp_cur(const MatrixHandle& A, Index rank, std::uint64_t seed);

}  // namespace itercur

// GPU test of the C++ facade (include/itercur/driver_b200.hpp), compiled by g++ against
// libitercur_facade.so and checked against the CPU oracle (liboracle.so, test infrastructure).
// Restates proj/tests/test_driver.cpp-style checks through itercur::iterative_cur:
// identical I/J/status and error to the oracle, the IterationObserver after every iteration,
// per-method pivot floors, the core's solves, and the reference's exception classes/messages.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "itercur/driver_b200.hpp"
#include "itercur_oracle.h"

using namespace itercur;

static int g_fail = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (!(cond)) {                                                          \
      std::fprintf(stderr, "CHECK failed at line %d: %s\n", __LINE__, #cond); \
      ++g_fail;                                                             \
    }                                                                       \
  } while (0)

template <class E, class F>
static bool throws_with(F&& f, const char* needle) {
  try {
    f();
  } catch (const E& e) {
    return std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

// low rank + relative noise, from the reference tests' mt19937_64 fixtures (oracles.hpp:30-37)
static DenseMatrix low_rank_plus_noise(Index m, Index n, Index r, double rel_noise, unsigned seed) {
  std::vector<double> x(m * r), y(n * r), g(m * n);
  oracle_fixture_random_gaussian(m, r, seed, x.data());
  oracle_fixture_random_gaussian(n, r, seed + 1, y.data());
  oracle_fixture_random_gaussian(m, n, seed + 2, g.data());
  DenseMatrix a(m, n);
  double sa = 0.0, sg = 0.0;
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) {
      double s = 0.0;
      for (Index k = 0; k < r; ++k) s += x[i + k * m] * y[j + k * n];
      a(i, j) = s;
      sa += s * s;
      sg += g[i + j * m] * g[i + j * m];
    }
  const double scale = rel_noise * std::sqrt(sa / sg);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < m; ++i) a(i, j) += scale * g[i + j * m];
  return a;
}

struct OracleRun {
  std::vector<int64_t> I, J;
  int status = 0;
  int64_t iters = 0;
};

static OracleRun oracle_run(const DenseMatrix& a, double eps, Index b, uint64_t seed, double floor) {
  oracle_config c{};
  c.epsilon = eps;
  c.b = b;
  c.alpha = 0.05;
  c.pivot_floor = floor;
  c.seed = seed;
  c.sparse_nnz = 8;
  const int64_t cap = std::min(a.rows(), a.cols());
  OracleRun o;
  o.I.assign(cap, 0);
  o.J.assign(cap, 0);
  std::vector<double> rhos(cap + 2);
  std::vector<int64_t> widths(cap + 2);
  oracle_result res{};
  res.cap_rank = cap;
  res.row_indices = o.I.data();
  res.col_indices = o.J.data();
  res.cap_iters = cap + 2;
  res.rhos = rhos.data();
  res.widths = widths.data();
  if (oracle_iterative_cur(a.data(), a.rows(), a.cols(), a.rows(), &c, &res) != 0) {
    std::fprintf(stderr, "oracle failed: %s\n", oracle_last_error());
    std::exit(2);
  }
  o.I.resize(res.rank);
  o.J.resize(res.rank);
  o.status = res.status;
  o.iters = res.n_iters;
  return o;
}

int main() {
  // ---- 1. parity with the oracle, observer after every iteration ----
  const DenseMatrix a = low_rank_plus_noise(400, 300, 40, 1e-9, 5);
  const MatrixHandle A(a);
  StoppingConfig cfg;
  cfg.epsilon = 1e-7;
  cfg.b = 8;
  SelectionMethod lupp;
  int calls = 0;
  Index last_rank = 0;
  bool observer_ok = true;
  auto observer = [&](const CurFactors& f, const IterationRecord& rec) {
    ++calls;
    observer_ok &= rec.k == calls - 1 && f.rank() == last_rank + rec.cols_added && rec.cols_added > 0;
    last_rank = f.rank();
    // C = A(:, J) and R = A(I, :) exactly, core = A(I, J)^{-1}
    const DenseMatrix& C = f.C.dense_data();
    const DenseMatrix& R = f.R.dense_data();
    for (Index q = 0; q < f.rank(); ++q) {
      for (Index i = 0; i < a.rows(); ++i) observer_ok &= C(i, q) == a(i, f.col_indices[q]);
      for (Index j = 0; j < a.cols(); ++j) observer_ok &= R(q, j) == a(f.row_indices[q], j);
    }
    DenseMatrix X(f.rank(), f.rank());
    for (Index q = 0; q < f.rank(); ++q)
      for (Index p = 0; p < f.rank(); ++p) X(p, q) = a(f.row_indices[p], f.col_indices[q]);
    const DenseMatrix Y = f.core.solve(X);
    double dev = 0.0;
    for (Index q = 0; q < f.rank(); ++q)
      for (Index p = 0; p < f.rank(); ++p) dev = std::max(dev, std::abs(Y(p, q) - (p == q ? 1.0 : 0.0)));
    observer_ok &= dev < 1e-6;
  };
  const CurResult res = iterative_cur(A, cfg, lupp, lupp, 3, observer);
  const OracleRun o = oracle_run(a, cfg.epsilon, cfg.b, 3, 1e-13);
  CHECK(res.factors.row_indices == o.I);
  CHECK(res.factors.col_indices == o.J);
  CHECK(static_cast<int>(res.trace.status) == o.status);
  CHECK(static_cast<int64_t>(res.trace.iterations.size()) == o.iters);
  CHECK(calls == static_cast<int>(res.trace.iterations.size()) && calls > 1);
  CHECK(observer_ok);
  CHECK(std::string(to_string(res.trace.status)) == "Converged");
  CHECK(res.trace.iterations.back().rho == res.trace.final_rho);

  // ---- 2. true_relative_error on the given matrix vs the oracle ----
  const double err = true_relative_error(A, res.factors);
  double err_o = 0.0;
  CHECK(oracle_true_relative_error(a.data(), a.rows(), a.cols(), a.rows(), o.I.data(), o.J.data(),
                                   static_cast<int64_t>(o.I.size()), &err_o) == 0);
  CHECK(std::abs(err - err_o) <= 1e-8);
  // a different matrix of the same shape gives a different error (the given A is honoured)
  DenseMatrix a2 = a;
  for (Index i = 0; i < a2.rows(); ++i) a2(i, 0) += 1.0;
  CHECK(true_relative_error(MatrixHandle(a2), res.factors) > 10 * err);
  CHECK(throws_with<std::invalid_argument>([&] { true_relative_error(MatrixHandle(DenseMatrix(3, 3)), res.factors); },
                                           "factors are for"));

  // ---- 3. the core: solve / solve_transposed / materialize against A(I, J) ----
  const Index r = res.factors.rank();
  DenseMatrix X(r, r), Xt(r, r);
  for (Index q = 0; q < r; ++q)
    for (Index p = 0; p < r; ++p) {
      X(p, q) = a(res.factors.row_indices[p], res.factors.col_indices[q]);
      Xt(q, p) = X(p, q);
    }
  const DenseMatrix P = res.factors.core.solve(X), Pt = res.factors.core.solve_transposed(Xt);
  const DenseMatrix M = res.factors.core.materialize();
  double dev = 0.0, devt = 0.0, devm = 0.0;
  for (Index q = 0; q < r; ++q)
    for (Index p = 0; p < r; ++p) {
      dev = std::max(dev, std::abs(P(p, q) - (p == q ? 1.0 : 0.0)));
      devt = std::max(devt, std::abs(Pt(p, q) - (p == q ? 1.0 : 0.0)));
      double mx = 0.0;  // (materialize() * X)(p, q)
      for (Index k = 0; k < r; ++k) mx += M(p, k) * X(k, q);
      devm = std::max(devm, std::abs(mx - (p == q ? 1.0 : 0.0)));
    }
  CHECK(dev < 1e-6 && devt < 1e-6 && devm < 1e-6);
  CHECK(throws_with<std::invalid_argument>([&] { res.factors.core.solve(DenseMatrix(r + 1, 2)); }, "apply_pinv_left"));
  CHECK(res.factors.C.rows() == a.rows() && res.factors.C.cols() == r && res.factors.R.rows() == r);

  // ---- 4. per-method pivot floors: a high row floor truncates row blocks only ----
  SelectionMethod strict_rows;
  strict_rows.pivot_floor = 0.99;
  const CurResult rs = iterative_cur(A, cfg, lupp, strict_rows, 3);
  CHECK(rs.trace.iterations.front().row_truncated && !rs.trace.iterations.front().col_truncated);
  SelectionMethod bad;
  bad.pivot_floor = 1.5;
  CHECK(throws_with<std::invalid_argument>([&] { iterative_cur(A, cfg, lupp, bad, 3); }, "pivot_floor"));

  // ---- 5. the reference's exception classes and messages ----
  CHECK(throws_with<std::invalid_argument>([&] { iterative_cur(MatrixHandle(DenseMatrix(4, 4)), cfg, lupp, lupp, 0); },
                                           "nonzero"));
  StoppingConfig big = cfg;
  big.b = 500;
  CHECK(throws_with<std::invalid_argument>([&] { iterative_cur(A, big, lupp, lupp, 0); }, "block exceeds row count"));
  SelectionMethod osinsky;
  osinsky.kind = PivotKind::Osinsky;
  CHECK(throws_with<std::runtime_error>([&] { iterative_cur(A, cfg, osinsky, lupp, 0); }, "not implemented"));
  StoppingConfig risky = cfg;
  risky.b = 2;
  risky.alpha = 0.1;
  risky.risk_adjust = true;
  CHECK(throws_with<std::domain_error>([&] { iterative_cur(A, risky, lupp, lupp, 0); }, "block too small"));
  DenseMatrix nan = a;
  nan(1, 1) = std::nan("");
  CHECK(throws_with<std::invalid_argument>([&] { MatrixHandle h(nan); }, "non-finite"));
  // an observer's exception propagates out of iterative_cur (the reference calls it inline)
  CHECK(throws_with<std::out_of_range>(
      [&] { iterative_cur(A, cfg, lupp, lupp, 3, [](const CurFactors&, const IterationRecord&) {
              throw std::out_of_range("observer says stop");
            }); },
      "observer says stop"));
  CHECK(std::abs(adjusted_threshold(1.0, 0.0, 1e-10, 100) - 1.0 / 4.98) < 5e-4 / 4.98);
  CHECK(std::abs(gratton_tail(4, std::sqrt(2.0)) - std::exp(-0.25)) < 1e-15);

  // ---- 6. CSR input and the s-LUPP baseline ----
  std::vector<Index> rp{0, 1, 3}, ci{2, 0, 1};
  std::vector<double> v{5.0, 1.0, -2.0};
  const MatrixHandle S(2, 3, rp, ci, v);
  CHECK(S.is_sparse() && S.nnz() == 3 && S.to_dense()(0, 2) == 5.0 && S.to_dense()(1, 1) == -2.0);
  CHECK(throws_with<std::out_of_range>([&] { MatrixHandle(2, 3, {0, 1, 1}, {3}, {1.0}); }, "out of range"));
  const CurFactors sl = slupp_cur(A, 25, 4);
  std::vector<int64_t> sI(25), sJ(25);
  int64_t srank = 0;
  CHECK(oracle_slupp_cur(a.data(), a.rows(), a.cols(), a.rows(), 25, 4, sI.data(), sJ.data(), &srank) == 0);
  sI.resize(srank);
  sJ.resize(srank);
  CHECK(sl.row_indices == sI && sl.col_indices == sJ);
  CHECK(throws_with<std::invalid_argument>([&] { slupp_cur(A, 301, 0); }, "rank must lie"));

  if (g_fail) {
    std::fprintf(stderr, "%d check(s) failed\n", g_fail);
    return 1;
  }
  std::printf("facade ok: rank %lld, %d observer calls, err %.3e (oracle %.3e)\n", static_cast<long long>(r), calls,
              err, err_o);
  return 0;
}

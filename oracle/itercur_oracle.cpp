// itercur_oracle.cpp — CPU ORACLE for the IterativeCUR hot path. TEST INFRASTRUCTURE.
//
// A plain-C++ (no Eigen: it is absent from this image) restatement of
// the reference algorithm, function by function, each citing the reference file:line
// it follows. Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// `--impl reference`) load this library; the product path never does.
//
// Dense matrices are column-major doubles, as in the reference (Eigen default;
// proj/src/matrix.cpp). Elementwise eliminations are written with separate
// multiply/subtract roundings (the reference Release build has no FMA,
// proj/CMakeLists.txt:1-9) and this file is compiled with -ffp-contract=off.
#include "itercur_oracle.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <thread>

namespace oracle {

// ---------------------------------------------------------------------------------
// Host threading for the CPU timing arm (no OpenMP runtime in this image): a persistent pool
// that splits an index range [b, e) into static contiguous chunks. Only loops over independent
// columns use it, each column's operations unchanged, so results are bitwise the 1-thread
// ones. ORACLE_THREADS (default: all hardware threads) sets the pool size; 1 = sequential.
// ---------------------------------------------------------------------------------
// Threads actually used per parallel loop (<= the pool size): oracle_set_threads() lowers it, so
// one process can time the same oracle on 1 core and on all cores.
std::atomic<int> g_thread_limit{1 << 30};

class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  int size() const { return std::min(nthreads_, g_thread_limit.load()); }
  void run(std::int64_t b, std::int64_t e, const std::function<void(std::int64_t)>& fn) {
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &fn;
    b_ = b;
    e_ = e;
    pending_ = nthreads_ - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    chunk(0, b, e, fn);  // the caller takes chunk 0
    lk.lock();
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() {
    const char* env = std::getenv("ORACLE_THREADS");
    int n = env ? std::atoi(env) : static_cast<int>(std::thread::hardware_concurrency());
    nthreads_ = n < 1 ? 1 : n;
    for (int t = 1; t < nthreads_; ++t) workers_.emplace_back([this, t] { loop(t); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void chunk(int t, std::int64_t b, std::int64_t e, const std::function<void(std::int64_t)>& fn) const {
    const int active = size();
    if (t >= active) return;
    const std::int64_t n = e - b, per = (n + active - 1) / active;
    const std::int64_t lo = b + t * per, hi = std::min(e, lo + per);
    for (std::int64_t i = lo; i < hi; ++i) fn(i);
  }
  void loop(int t) {
    std::uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      const auto* fn = fn_;
      const std::int64_t b = b_, e = e_;
      lk.unlock();
      chunk(t, b, e, *fn);
      lk.lock();
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  int nthreads_ = 1;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(std::int64_t)>* fn_ = nullptr;
  std::int64_t b_ = 0, e_ = 0;
  int pending_ = 0;
  std::uint64_t gen_ = 0;
  bool stop_ = false;
};

template <class F>
void parallel_for(std::int64_t b, std::int64_t e, bool worth_it, F&& f) {
  if (e <= b) return;
  Pool* pool = worth_it && (e - b) > 1 ? &Pool::get() : nullptr;
  if (!pool || pool->size() == 1) {
    for (std::int64_t i = b; i < e; ++i) f(i);
    return;
  }
  const std::function<void(std::int64_t)> fn = [&](std::int64_t i) { f(i); };
  pool->run(b, e, fn);
}

using Index = std::int64_t;
using IndexList = std::vector<Index>;

struct Mat {
  Index rows = 0, cols = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(Index r, Index c) : rows(r), cols(c), v(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(Index i, Index j) { return v[static_cast<size_t>(i + j * rows)]; }
  double operator()(Index i, Index j) const { return v[static_cast<size_t>(i + j * rows)]; }
  double* col(Index j) { return v.data() + j * rows; }
  const double* col(Index j) const { return v.data() + j * rows; }
  bool empty() const { return rows == 0 || cols == 0; }
};

// Plain sequential sum of squares (Eigen's squaredNorm order differs; ulp-level only).
double sq_norm(const double* p, Index count) {
  double s = 0.0;
  for (Index k = 0; k < count; ++k) s += p[k] * p[k];
  return s;
}
double fro_norm(const Mat& a) { return std::sqrt(sq_norm(a.v.data(), static_cast<Index>(a.v.size()))); }

// ---------------------------------------------------------------------------------
// rng — proj/src/rng.cpp
// ---------------------------------------------------------------------------------
constexpr std::uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;   // rng.cpp:9-10
constexpr std::uint32_t kWeyl0 = 0x9E3779B9u, kWeyl1 = 0xBB67AE85u; // rng.cpp:11-12

// rng.cpp:30-43 (Random123 Philox4x32-10 round)
std::array<std::uint32_t, 4> philox(std::array<std::uint32_t, 4> ctr, std::array<std::uint32_t, 2> key) {
  for (int round = 0; round < 10; ++round) {
    const std::uint64_t p0 = static_cast<std::uint64_t>(kMul0) * ctr[0];
    const std::uint64_t p1 = static_cast<std::uint64_t>(kMul1) * ctr[2];
    ctr = {static_cast<std::uint32_t>(p1 >> 32) ^ ctr[1] ^ key[0], static_cast<std::uint32_t>(p1),
           static_cast<std::uint32_t>(p0 >> 32) ^ ctr[3] ^ key[1], static_cast<std::uint32_t>(p0)};
    key[0] += kWeyl0;
    key[1] += kWeyl1;
  }
  return ctr;
}
// rng.cpp:14-18
inline double to_unit(std::uint32_t hi, std::uint32_t lo) {
  const std::uint64_t bits = (static_cast<std::uint64_t>(hi) << 32) | lo;
  return (static_cast<double>(bits >> 11) + 0.5) * 0x1p-53;
}
// rng.cpp:20-26
inline std::array<std::uint32_t, 4> counter_for(std::uint32_t stream, Index i, Index j) {
  return {stream, static_cast<std::uint32_t>(i), static_cast<std::uint32_t>(j),
          static_cast<std::uint32_t>((static_cast<std::uint64_t>(i) >> 32) ^
                                     ((static_cast<std::uint64_t>(j) >> 32) << 8))};
}
inline std::array<std::uint32_t, 2> key_for(std::uint64_t seed) {
  return {static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32)};
}
// rng.cpp:45-52 — cosine branch of Box-Muller, evaluation order kept.
double normal_at(std::uint64_t seed, std::uint32_t stream, Index i, Index j) {
  const auto r = philox(counter_for(stream, i, j), key_for(seed));
  const double u1 = to_unit(r[0], r[1]);
  const double u2 = to_unit(r[2], r[3]);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}
// rng.cpp:54-59
double uniform_at(std::uint64_t seed, std::uint32_t stream, Index i, Index j) {
  const auto r = philox(counter_for(stream, i, j), key_for(seed));
  return to_unit(r[0], r[1]);
}
// rng.cpp:61-67
Mat gaussian_matrix(Index rows, Index cols, std::uint64_t seed, std::uint32_t stream) {
  Mat out(rows, cols);
  parallel_for(0, cols, rows * cols > 65536, [&](Index j) {  // entries are independent of fill order
    for (Index i = 0; i < rows; ++i) out(i, j) = normal_at(seed, stream, i, j);
  });
  return out;
}

// Sparse-sign stream — NEW (the reference has none). Column i of
// Omega (= row i of A) gets zeta_eff = min(zeta, c) distinct destination rows drawn by a
// partial Fisher-Yates over [0, c), one Philox block per slot t:
//   r = philox(counter_for(7, i, t), key(seed)); j_t = t + floor(r0 * (c - t) / 2^32);
//   swap(perm[t], perm[j_t]); h_t = perm[t]; sign = (r1 & 1) ? -1 : +1.
// Omega(h_t, i) = sign / sqrt(zeta_eff); the scale is applied once per output entry.
void sparse_sign_column(std::uint64_t seed, Index i, Index c, int zeta_eff, std::int32_t* rows,
                        std::int8_t* signs) {
  std::int32_t pos[64], val[64];  // partial-permutation overrides (<= zeta_eff entries)
  int nover = 0;
  auto get = [&](std::int32_t p) {
    for (int q = 0; q < nover; ++q)
      if (pos[q] == p) return val[q];
    return p;
  };
  auto set = [&](std::int32_t p, std::int32_t v) {
    for (int q = 0; q < nover; ++q)
      if (pos[q] == p) { val[q] = v; return; }
    pos[nover] = p; val[nover] = v; ++nover;
  };
  const auto key = key_for(seed);
  for (int t = 0; t < zeta_eff; ++t) {
    const auto r = philox(counter_for(ORACLE_STREAM_SPARSE_SIGN, i, t), key);
    const std::uint64_t span = static_cast<std::uint64_t>(c - t);
    const std::int32_t jt = t + static_cast<std::int32_t>((static_cast<std::uint64_t>(r[0]) * span) >> 32);
    const std::int32_t vt = get(t), vj = get(jt);
    set(t, vj);
    set(jt, vt);
    rows[t] = vj;
    signs[t] = (r[1] & 1u) ? -1 : 1;
  }
}

// ---------------------------------------------------------------------------------
// Complete orthogonal decomposition — restates Eigen's CompleteOrthogonalDecomposition
// as used by proj/src/pinv.cpp:45-65 (ColPivHouseholderQR with threshold, then the
// minimum-norm least-squares solve). Eigen itself is not in the image; this follows
// its documented algorithm (pivot = largest updated column norm, LAPACK-style norm
// downdating, rank = #{|R_ii| > threshold * max pivot}).
// ---------------------------------------------------------------------------------
struct Cod {
  Index rows = 0, cols = 0, rank = 0;
  Mat qr;                      // Householder vectors below the diagonal, R on/above
  std::vector<double> hcoeffs; // tau per reflector
  std::vector<Index> perm;     // column k of QR = column perm[k] of X
  double maxpivot = 0.0;
  // For rank < cols: QR of [R11 R12]^T (cols x rank) giving the minimum-norm solve.
  Mat lq;
  std::vector<double> lq_tau;

  static void make_householder(double* x, Index len, double& tau, double& beta) {
    // Eigen MatrixBase::makeHouseholder: x = [c0; tail]
    const double tiny = std::numeric_limits<double>::min();
    const double c0 = x[0];
    double tail_sq = 0.0;
    for (Index k = 1; k < len; ++k) tail_sq += x[k] * x[k];
    if (tail_sq <= tiny) {
      tau = 0.0;
      beta = c0;
      for (Index k = 1; k < len; ++k) x[k] = 0.0;
    } else {
      beta = std::sqrt(c0 * c0 + tail_sq);
      if (c0 >= 0.0) beta = -beta;
      for (Index k = 1; k < len; ++k) x[k] = x[k] / (c0 - beta);
      tau = (beta - c0) / beta;
    }
  }
  // apply H = I - tau [1; v][1; v]^T from the left to column y (length len)
  static void apply_left(const double* v, Index len, double tau, double* y) {
    if (tau == 0.0) return;
    double tmp = y[0];
    for (Index k = 1; k < len; ++k) tmp += v[k] * y[k];
    y[0] -= tau * tmp;
    for (Index k = 1; k < len; ++k) y[k] -= tau * v[k] * tmp;
  }

  void compute(const Mat& x, double threshold) {
    rows = x.rows;
    cols = x.cols;
    qr = x;
    const Index size = std::min(rows, cols);
    hcoeffs.assign(static_cast<size_t>(size), 0.0);
    perm.resize(static_cast<size_t>(cols));
    for (Index j = 0; j < cols; ++j) perm[static_cast<size_t>(j)] = j;
    std::vector<double> norm_upd(static_cast<size_t>(cols)), norm_dir(static_cast<size_t>(cols));
    for (Index j = 0; j < cols; ++j) norm_dir[static_cast<size_t>(j)] = norm_upd[static_cast<size_t>(j)] =
        std::sqrt(sq_norm(qr.col(j), rows));
    const double downdate_thr = std::sqrt(std::numeric_limits<double>::epsilon());
    maxpivot = 0.0;
    for (Index k = 0; k < size; ++k) {
      Index best = k;
      for (Index j = k + 1; j < cols; ++j)
        if (norm_upd[static_cast<size_t>(j)] > norm_upd[static_cast<size_t>(best)]) best = j;
      if (best != k) {
        std::swap_ranges(qr.col(k), qr.col(k) + rows, qr.col(best));
        std::swap(norm_upd[static_cast<size_t>(k)], norm_upd[static_cast<size_t>(best)]);
        std::swap(norm_dir[static_cast<size_t>(k)], norm_dir[static_cast<size_t>(best)]);
        std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(best)]);
      }
      double tau = 0.0, beta = 0.0;
      make_householder(qr.col(k) + k, rows - k, tau, beta);
      qr(k, k) = beta;
      hcoeffs[static_cast<size_t>(k)] = tau;
      maxpivot = std::max(maxpivot, std::abs(beta));
      // columns are independent: threads change nothing but the wall time (same operations, same order)
      parallel_for(k + 1, cols, (cols - k) * (rows - k) > 32768, [&](Index j) {
        // apply reflector (stored with implicit leading 1) to column j
        double* y = qr.col(j) + k;
        const double* v = qr.col(k) + k;
        if (tau != 0.0) {
          double tmp = y[0];
          for (Index q = 1; q < rows - k; ++q) tmp += v[q] * y[q];
          y[0] -= tau * tmp;
          for (Index q = 1; q < rows - k; ++q) y[q] -= tau * v[q] * tmp;
        }
      });
      parallel_for(k + 1, cols, (cols - k) * (rows - k) > 32768, [&](Index j) {
        double& nu = norm_upd[static_cast<size_t>(j)];
        if (nu != 0.0) {
          double temp = std::abs(qr(k, j)) / nu;
          temp = (1.0 + temp) * (1.0 - temp);
          if (temp < 0.0) temp = 0.0;
          const double ratio = nu / norm_dir[static_cast<size_t>(j)];
          const double temp2 = temp * ratio * ratio;
          if (temp2 <= downdate_thr) {
            norm_dir[static_cast<size_t>(j)] = std::sqrt(sq_norm(qr.col(j) + k + 1, rows - k - 1));
            nu = norm_dir[static_cast<size_t>(j)];
          } else {
            nu *= std::sqrt(temp);
          }
        }
      });
    }
    const double pre = std::abs(maxpivot) * threshold;
    rank = 0;
    for (Index i = 0; i < size; ++i)
      if (std::abs(qr(i, i)) > pre) ++rank;
    lq = Mat();
    lq_tau.clear();
    if (rank < cols && rank > 0) {
      // Minimum-norm solve of [R11 R12] z = c: QR of its transpose (cols x rank).
      lq = Mat(cols, rank);
      for (Index i = 0; i < rank; ++i)
        for (Index j = i; j < cols; ++j) lq(j, i) = qr(i, j);
      lq_tau.assign(static_cast<size_t>(rank), 0.0);
      for (Index k = 0; k < rank; ++k) {
        double tau = 0.0, beta = 0.0;
        make_householder(lq.col(k) + k, cols - k, tau, beta);
        lq(k, k) = beta;
        lq_tau[static_cast<size_t>(k)] = tau;
        parallel_for(k + 1, rank, (rank - k) * (cols - k) > 32768,
                     [&](Index j) { apply_left(lq.col(k) + k, cols - k, tau, lq.col(j) + k); });
      }
    }
  }

  // X^+ * rhs (rows x k) -> cols x k; minimum-norm least squares.
  Mat solve(const Mat& rhs) const {
    if (rhs.rows != rows) throw std::invalid_argument("apply_pinv_left: expected " + std::to_string(rows) +
                                                      " rows, got " + std::to_string(rhs.rows));
    Mat out(cols, rhs.cols);
    parallel_for(0, rhs.cols, rhs.cols * rows * cols > 65536, [&](Index col) {
      std::vector<double> c(static_cast<size_t>(rows)), z(static_cast<size_t>(cols));
      std::copy(rhs.col(col), rhs.col(col) + rows, c.begin());
      const Index size = std::min(rows, cols);
      for (Index k = 0; k < size; ++k)  // c = Q^T b
        apply_left(qr.col(k) + k, rows - k, hcoeffs[static_cast<size_t>(k)], c.data() + k);
      std::fill(z.begin(), z.end(), 0.0);
      if (rank == cols) {
        for (Index i = rank - 1; i >= 0; --i) {  // back substitution with R11
          double s = c[static_cast<size_t>(i)];
          for (Index j = i + 1; j < rank; ++j) s -= qr(i, j) * z[static_cast<size_t>(j)];
          z[static_cast<size_t>(i)] = s / qr(i, i);
        }
      } else if (rank > 0) {
        // [R11 R12] = (Q2 R2)^T with R2 = upper triangle of lq: solve R2^T w = c, z = Q2 [w; 0]
        std::vector<double> w(static_cast<size_t>(cols), 0.0);
        for (Index i = 0; i < rank; ++i) {
          double s = c[static_cast<size_t>(i)];
          for (Index j = 0; j < i; ++j) s -= lq(j, i) * w[static_cast<size_t>(j)];
          w[static_cast<size_t>(i)] = s / lq(i, i);
        }
        for (Index k = rank - 1; k >= 0; --k)
          apply_left(lq.col(k) + k, cols - k, lq_tau[static_cast<size_t>(k)], w.data() + k);
        for (Index j = 0; j < cols; ++j) z[static_cast<size_t>(j)] = w[static_cast<size_t>(j)];
      }
      for (Index k = 0; k < cols; ++k) out(perm[static_cast<size_t>(k)], col) = z[static_cast<size_t>(k)];
    });
    return out;
  }
};

// proj/include/itercur/pinv.hpp:16-40, proj/src/pinv.cpp:11-65
struct FactoredPinv {
  bool valid = false;
  Cod cod, cod_t;
  double tol = 0.0;
};
Mat transpose(const Mat& a) {
  Mat t(a.cols, a.rows);
  for (Index j = 0; j < a.cols; ++j)
    for (Index i = 0; i < a.rows; ++i) t(j, i) = a(i, j);
  return t;
}
FactoredPinv build_pinv(const Mat& x, double tol = -1.0) {
  if (x.empty()) throw std::invalid_argument("build_pinv: empty matrix");
  if (fro_norm(x) == 0.0) throw std::runtime_error("singular cross block");  // pinv.cpp:49
  FactoredPinv p;
  p.valid = true;
  p.tol = tol >= 0.0 ? tol : 1e-12 * static_cast<double>(std::max(x.rows, x.cols));  // pinv.cpp:54
  p.cod.compute(x, p.tol);                                                          // pinv.cpp:56-58
  p.cod_t.compute(transpose(x), p.tol);                                             // pinv.cpp:59-60
  return p;
}

// ---------------------------------------------------------------------------------
// dense matrix helpers — proj/src/matrix.cpp (dense paths only)
// ---------------------------------------------------------------------------------
[[noreturn]] void bad_index(const char* where, Index idx, Index bound) {  // matrix.cpp:19-22
  throw std::out_of_range(std::string(where) + ": index " + std::to_string(idx) + " out of range [0, " +
                          std::to_string(bound) + ")");
}
struct View {  // non-owning column-major view of the input
  const double* p;
  Index rows, cols, ld;
  double operator()(Index i, Index j) const { return p[i + j * ld]; }
};
Mat gather_cols(const View& a, const IndexList& cols) {  // matrix.cpp:134-144
  for (Index j : cols)
    if (j < 0 || j >= a.cols) bad_index("gather_cols", j, a.cols);
  Mat out(a.rows, static_cast<Index>(cols.size()));
  for (size_t k = 0; k < cols.size(); ++k)
    std::memcpy(out.col(static_cast<Index>(k)), a.p + cols[k] * a.ld, sizeof(double) * a.rows);
  return out;
}
Mat gather_rows(const View& a, const IndexList& rows) {  // matrix.cpp:196-206
  for (Index i : rows)
    if (i < 0 || i >= a.rows) bad_index("gather_rows", i, a.rows);
  Mat out(static_cast<Index>(rows.size()), a.cols);
  parallel_for(0, a.cols, a.cols * static_cast<Index>(rows.size()) > 65536, [&](Index j) {
    for (size_t k = 0; k < rows.size(); ++k) out(static_cast<Index>(k), j) = a(rows[k], j);
  });
  return out;
}
View view(const Mat& m) { return View{m.v.data(), m.rows, m.cols, m.rows}; }
// C += alpha * A * B (plain loops, column-major; order a-priori fixed)
void gemm_acc(const Mat& a, const Mat& b, Mat& c, double alpha) {
  parallel_for(0, b.cols, b.cols * a.cols * a.rows > 65536, [&](Index j) {
    for (Index k = 0; k < a.cols; ++k) {
      const double bk = alpha * b(k, j);
      if (bk == 0.0) continue;
      const double* ak = a.col(k);
      double* cj = c.col(j);
      for (Index i = 0; i < a.rows; ++i) cj[i] += ak[i] * bk;
    }
  });
}

// proj/include/itercur/pinv.hpp:57-66
struct CurFactors {
  IndexList I, J;
  Mat C, R;
  FactoredPinv core;
  bool empty() const { return J.empty(); }
  Index rank() const { return static_cast<Index>(J.size()); }
};
void check_distinct(const IndexList& idx, const char* what) {  // pinv.cpp:86-91
  std::unordered_set<Index> seen;
  for (Index i : idx)
    if (!seen.insert(i).second) throw std::invalid_argument(std::string(what) + " indices must be distinct");
}
// proj/src/pinv.cpp:94-111
CurFactors make_cur_factors(const View& a, IndexList I, IndexList J, double tol = -1.0) {
  if (I.size() != J.size()) throw std::invalid_argument("cross block must be square: |I| != |J|");
  check_distinct(I, "row");
  check_distinct(J, "column");
  CurFactors cur;
  if (I.empty()) return cur;
  for (Index i : I)
    if (i < 0 || i >= a.rows) bad_index("gather_rows", i, a.rows);
  for (Index j : J)
    if (j < 0 || j >= a.cols) bad_index("gather_cols", j, a.cols);
  Mat cross(static_cast<Index>(I.size()), static_cast<Index>(J.size()));  // gather_block, matrix.cpp:224-227
  for (size_t q = 0; q < J.size(); ++q)
    for (size_t p = 0; p < I.size(); ++p) cross(static_cast<Index>(p), static_cast<Index>(q)) = a(I[p], J[q]);
  cur.core = build_pinv(cross, tol);
  cur.C = gather_cols(a, J);
  cur.R = gather_rows(a, I);
  cur.I = std::move(I);
  cur.J = std::move(J);
  return cur;
}
// apply_pinv_left / right, pinv.cpp:67-81
Mat apply_pinv_left(const FactoredPinv& p, const Mat& m) { return p.cod.solve(m); }
Mat apply_pinv_right(const FactoredPinv& p, const Mat& m) { return transpose(p.cod_t.solve(transpose(m))); }

// ---------------------------------------------------------------------------------
// sketch — proj/include/itercur/sketch.hpp, proj/src/sketch.cpp
// ---------------------------------------------------------------------------------
inline Index sketch_rows_for_block(Index b) { return (11 * b) / 10; }  // sketch.hpp:10

// ||A||_F^2 as per-column partial sums added in column order (threads split the columns, so the
// value does not depend on the thread count); optionally the MatrixHandle finite check
// (matrix.cpp:73-77).
double column_sumsq(const View& a, bool check_finite) {
  std::vector<double> part(static_cast<size_t>(std::max<Index>(a.cols, 0)), 0.0);
  std::atomic<bool> bad{false};
  parallel_for(0, a.cols, a.cols * a.rows > 65536, [&](Index j) {
    const double* aj = a.p + j * a.ld;
    double s = 0.0;
    bool fin = true;
    for (Index i = 0; i < a.rows; ++i) {
      fin &= std::isfinite(aj[i]);
      s += aj[i] * aj[i];
    }
    if (check_finite && !fin) bad.store(true);
    part[static_cast<size_t>(j)] = s;
  });
  if (bad.load()) throw std::invalid_argument("matrix contains non-finite entries");
  double asq = 0.0;
  for (double v : part) asq += v;
  return asq;
}

struct SketchState {  // sketch.hpp:19-27
  Mat sketched_input;  // S*A (c x n)
  Mat col_residual;    // Y
  double ga_norm = 0.0;
  double a_norm = 0.0;
  Index c = 0, b = 0;
};

// make_sketch, sketch.cpp:10-24 — plus the new sparse-sign kind. ||A|| is computed in the
// same pass (the reference's separate fro_norm(A) zero check, driver.cpp:52).
SketchState make_sketch(std::uint64_t seed, Index b, const View& a, int kind, int zeta) {
  if (b < 1) throw std::invalid_argument("block size must be at least 1");
  if (a.rows == 0 || a.cols == 0) throw std::invalid_argument("matrix must be nonempty");
  if (b > a.rows) throw std::invalid_argument("block exceeds row count");
  SketchState st;
  st.b = b;
  st.c = sketch_rows_for_block(b);
  const Index c = st.c, m = a.rows, n = a.cols;
  st.sketched_input = Mat(c, n);
  double asq = 0.0;
  if (kind == ORACLE_SKETCH_GAUSSIAN) {
    const Mat g = gaussian_matrix(c, m, seed, ORACLE_STREAM_SKETCH);  // sketch.cpp:19
    asq = column_sumsq(a, false);
    parallel_for(0, n, n * m * c > 65536, [&](Index j) {  // sketch.cpp:20 (G*A)
      double* y = st.sketched_input.col(j);
      const double* aj = a.p + j * a.ld;
      for (Index k = 0; k < m; ++k) {
        const double akj = aj[k];
        const double* gk = g.col(k);
        for (Index i = 0; i < c; ++i) y[i] += gk[i] * akj;
      }
    });
  } else if (kind == ORACLE_SKETCH_SPARSE_SIGN) {
    const int zeta_eff = static_cast<int>(std::min<Index>(zeta, c));
    if (zeta_eff < 1) throw std::invalid_argument("sparse_nnz must be at least 1");
    std::vector<std::int32_t> rows(static_cast<size_t>(m * zeta_eff));
    std::vector<std::int8_t> signs(static_cast<size_t>(m * zeta_eff));
    for (Index i = 0; i < m; ++i)
      sparse_sign_column(seed, i, c, zeta_eff, rows.data() + i * zeta_eff, signs.data() + i * zeta_eff);
    const double scale = 1.0 / std::sqrt(static_cast<double>(zeta_eff));
    asq = column_sumsq(a, false);
    // Y(h, j) = scale * sum over rows i in ascending order of sign * A(i, j) for the rows i that
    // hit h. Walked per sketch row h over its (ascending) row list, the additions into each Y(h, j)
    // happen in exactly the order of the row-major scatter "for i: y[h_t(i)] +-= A(i, j)", so the
    // result is bitwise that loop's — without its store-to-load dependency chains through y.
    std::vector<std::vector<std::int32_t>> hits(static_cast<size_t>(c));  // i, or ~i for a negative sign
    for (Index i = 0; i < m; ++i)
      for (int t = 0; t < zeta_eff; ++t) {
        const size_t q = static_cast<size_t>(i * zeta_eff + t);
        hits[static_cast<size_t>(rows[q])].push_back(signs[q] > 0 ? static_cast<std::int32_t>(i)
                                                                  : ~static_cast<std::int32_t>(i));
      }
    parallel_for(0, n, n * m > 65536, [&](Index j) {
      double* y = st.sketched_input.col(j);
      const double* aj = a.p + j * a.ld;
      for (Index h = 0; h < c; ++h) {
        double s = 0.0;
        for (const std::int32_t e : hits[static_cast<size_t>(h)]) {
          // branch-free s -/+= A(i, j): x - y is x + (-y) exactly in IEEE arithmetic
          const std::int32_t i = e ^ (e >> 31);
          std::uint64_t bits;
          std::memcpy(&bits, aj + i, sizeof bits);
          bits ^= static_cast<std::uint64_t>(static_cast<std::uint32_t>(e) >> 31) << 63;
          double v;
          std::memcpy(&v, &bits, sizeof v);
          s += v;
        }
        y[h] = s * scale;
      }
    });
  } else {
    throw std::invalid_argument("unknown sketch kind");
  }
  st.a_norm = std::sqrt(asq);
  st.col_residual = st.sketched_input;
  st.ga_norm = fro_norm(st.sketched_input);  // sketch.cpp:22
  return st;
}

// downdate_col_residual, sketch.cpp:26-41
double downdate_col_residual(SketchState& st, const CurFactors& cur) {
  if (cur.empty()) {
    st.col_residual = st.sketched_input;
    return st.ga_norm > 0.0 ? 1.0 : 0.0;
  }
  const Index r = cur.rank();
  Mat gc(st.c, r);
  for (Index k = 0; k < r; ++k)
    std::memcpy(gc.col(k), st.sketched_input.col(cur.J[static_cast<size_t>(k)]), sizeof(double) * st.c);
  const Mat gcu = apply_pinv_right(cur.core, gc);  // c x r
  st.col_residual = st.sketched_input;
  gemm_acc(gcu, cur.R, st.col_residual, -1.0);
  return st.ga_norm > 0.0 ? fro_norm(st.col_residual) / st.ga_norm : 0.0;
}

// row_residual, sketch.cpp:43-60
Mat row_residual(const View& a, const CurFactors& cur, const IndexList& new_cols) {
  if (!cur.empty()) {
    std::unordered_set<Index> held(cur.J.begin(), cur.J.end());
    for (Index j : new_cols)
      if (held.count(j)) throw std::invalid_argument("row_residual: column " + std::to_string(j) + " already selected");
  }
  Mat out = gather_cols(a, new_cols);
  if (cur.empty()) return out;
  const Mat r_cols = gather_cols(view(cur.R), new_cols);
  const Mat core_r = apply_pinv_left(cur.core, r_cols);
  gemm_acc(cur.C, core_r, out, -1.0);
  return out;
}

// ---------------------------------------------------------------------------------
// selection — proj/src/select.cpp
// ---------------------------------------------------------------------------------
constexpr double kAbsFloorFactor = 1e2 * std::numeric_limits<double>::epsilon();  // select.cpp:11

struct SelectionResult {  // select.hpp:17-21
  IndexList indices;
  bool truncated = false;
  double last_pivot_magnitude = 0.0;
  std::vector<double> best, second;  // per accepted step (oracle-only margin log)
};

std::vector<char> build_mask(Index size, const IndexList& exclude, const char* where) {  // select.cpp:13-22
  std::vector<char> banned(static_cast<size_t>(size), 0);
  for (Index e : exclude) {
    if (e < 0 || e >= size)
      throw std::out_of_range(std::string(where) + ": excluded index " + std::to_string(e) + " out of range");
    banned[static_cast<size_t>(e)] = 1;
  }
  return banned;
}

// lupp_pivot_rows, select.cpp:34-74. W is rows x cols column-major (a private copy).
SelectionResult lupp_pivot_rows(Mat w, Index b, double pivot_floor, double abs_floor, std::vector<char> banned) {
  SelectionResult res;
  const Index steps = std::min(b, w.cols);
  double first_pivot = 0.0;
  for (Index s = 0; s < steps; ++s) {
    Index best = -1;
    double best_mag = -1.0, second = -1.0;
    const double* ws = w.col(s);
    for (Index i = 0; i < w.rows; ++i) {
      if (banned[static_cast<size_t>(i)]) continue;
      const double mag = std::abs(ws[i]);
      if (mag > best_mag) {
        second = best_mag;
        best_mag = mag;
        best = i;
      } else if (mag > second) {
        second = mag;
      }
    }
    if (best < 0 || best_mag <= abs_floor) break;
    if (s == 0)
      first_pivot = best_mag;
    else if (best_mag < pivot_floor * first_pivot)
      break;
    res.indices.push_back(best);
    res.last_pivot_magnitude = best_mag;
    res.best.push_back(best_mag);
    res.second.push_back(second);
    banned[static_cast<size_t>(best)] = 1;
    if (s + 1 < w.cols) {
      const double pivot = w(best, s);
      for (Index t = s + 1; t < w.cols; ++t) {  // column-wise sweep; each entry updated once
        const double wb = w(best, t);
        double* wt = w.col(t);
        for (Index i = 0; i < w.rows; ++i) {
          if (banned[static_cast<size_t>(i)]) continue;
          const double factor = ws[i] / pivot;
          const double prod = factor * wb;
          wt[i] = wt[i] - prod;
        }
      }
    }
  }
  res.truncated = static_cast<Index>(res.indices.size()) < b;
  return res;
}

// qrcp_pivot_cols, select.cpp:79-117 (API surface; not on any BASELINE config)
SelectionResult qrcp_pivot_cols(Mat w, Index b, double pivot_floor, double abs_floor, std::vector<char> banned) {
  SelectionResult res;
  const Index steps = std::min(b, std::min(w.rows, w.cols));
  double first_pivot = 0.0;
  for (Index s = 0; s < steps; ++s) {
    Index best = -1;
    double best_sq = -1.0;
    for (Index j = 0; j < w.cols; ++j) {
      if (banned[static_cast<size_t>(j)]) continue;
      const double sq = sq_norm(w.col(j), w.rows);
      if (sq > best_sq) { best_sq = sq; best = j; }
    }
    if (best < 0) break;
    const double best_mag = std::sqrt(best_sq);
    if (best_mag <= abs_floor) break;
    if (s == 0) first_pivot = best_mag;
    else if (best_mag < pivot_floor * first_pivot) break;
    res.indices.push_back(best);
    res.last_pivot_magnitude = best_mag;
    res.best.push_back(best_mag);
    res.second.push_back(-1.0);
    banned[static_cast<size_t>(best)] = 1;
    std::vector<double> q(w.col(best), w.col(best) + w.rows);
    for (double& x : q) x /= best_mag;
    for (Index j = 0; j < w.cols; ++j) {
      if (banned[static_cast<size_t>(j)]) continue;
      double dot = 0.0;
      for (Index i = 0; i < w.rows; ++i) dot += q[static_cast<size_t>(i)] * w(i, j);
      for (Index i = 0; i < w.rows; ++i) w(i, j) -= q[static_cast<size_t>(i)] * dot;
    }
  }
  res.truncated = static_cast<Index>(res.indices.size()) < b;
  return res;
}

void validate(const Mat& m, double pivot_floor) {  // select.cpp:24-28
  if (!(pivot_floor > 0.0 && pivot_floor < 1.0)) throw std::invalid_argument("pivot_floor must lie in (0, 1)");
  for (double x : m.v)
    if (!std::isfinite(x)) throw std::invalid_argument("selection input must be finite");
}

// select_columns, select.cpp:121-139
SelectionResult select_columns(const Mat& m, Index b, int method, double pivot_floor, const IndexList& exclude) {
  validate(m, pivot_floor);
  if (b < 0 || b > m.rows)
    throw std::invalid_argument("select_columns: block size " + std::to_string(b) + " exceeds sketch rows " +
                                std::to_string(m.rows));
  const double abs_floor = kAbsFloorFactor * fro_norm(m);
  auto banned = build_mask(m.cols, exclude, "select_columns");
  switch (method) {
    case ORACLE_PIVOT_LUPP: return lupp_pivot_rows(transpose(m), b, pivot_floor, abs_floor, std::move(banned));
    case ORACLE_PIVOT_QRCP: return qrcp_pivot_cols(m, b, pivot_floor, abs_floor, std::move(banned));
    case ORACLE_PIVOT_OSINSKY: throw std::runtime_error("Osinsky selection not implemented");
  }
  throw std::logic_error("unknown selection method");
}
// select_rows, select.cpp:141-165
SelectionResult select_rows(const Mat& m, Index b, int method, double pivot_floor, const IndexList& exclude) {
  validate(m, pivot_floor);
  if (b < 0) throw std::invalid_argument("select_rows: negative block size");
  const Index effective = std::min(b, m.cols);
  const double abs_floor = kAbsFloorFactor * fro_norm(m);
  auto banned = build_mask(m.rows, exclude, "select_rows");
  switch (method) {
    case ORACLE_PIVOT_LUPP: {
      auto r = lupp_pivot_rows(m, effective, pivot_floor, abs_floor, std::move(banned));
      r.truncated = static_cast<Index>(r.indices.size()) < b;
      return r;
    }
    case ORACLE_PIVOT_QRCP: {
      auto r = qrcp_pivot_cols(transpose(m), effective, pivot_floor, abs_floor, std::move(banned));
      r.truncated = static_cast<Index>(r.indices.size()) < b;
      return r;
    }
    case ORACLE_PIVOT_OSINSKY: throw std::runtime_error("Osinsky selection not implemented");
  }
  throw std::logic_error("unknown selection method");
}

// ---------------------------------------------------------------------------------
// driver — proj/src/driver.cpp
// ---------------------------------------------------------------------------------
double adjusted_threshold(double epsilon, double delta, double alpha, Index c) {  // driver.cpp:28-39
  if (!(alpha > 0.0 && alpha < 1.0)) throw std::invalid_argument("alpha must lie in (0, 1)");
  if (delta < 0.0) throw std::invalid_argument("delta must be nonnegative");
  if (c < 1) throw std::invalid_argument("sketch rows must be positive");
  const double nla = -std::log(alpha);
  if (static_cast<double>(c) <= 4.0 * nla) throw std::domain_error("block too small for requested alpha");
  const double xi = (1.0 + delta) * std::sqrt(1.0 - 2.0 * std::sqrt(nla / static_cast<double>(c)));
  return xi * epsilon;
}
double gratton_tail(Index c, double tau) {  // driver.cpp:41-46
  if (c < 1) throw std::invalid_argument("sketch rows must be positive");
  if (!(tau > 1.0)) throw std::domain_error("tau must exceed 1");
  const double t2 = tau * tau;
  return std::exp(-static_cast<double>(c) * (t2 - 1.0) * (t2 - 1.0) / (4.0 * t2 * t2));
}

using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

void log_steps(oracle_result* res, int kind, Index k, const SelectionResult& sel) {
  for (size_t s = 0; s < sel.indices.size(); ++s) {
    const Index slot = res->n_steps++;
    if (slot < res->cap_steps) {
      res->step_kind[slot] = kind;
      res->step_iter[slot] = k;
      res->step_index[slot] = sel.indices[s];
      res->step_best[slot] = sel.best[s];
      res->step_second[slot] = sel.second[s];
    }
  }
}

// iterative_cur, driver.cpp:48-167
void iterative_cur(const View& a, const oracle_config& cfg, oracle_result* res) {
  // MatrixHandle construction rejects non-finite entries (matrix.cpp:73-77); then the
  // driver's validation order (driver.cpp:51-54).
  // (per-column partial sums, added in column order: the same value for any thread count)
  const double asq = column_sumsq(a, /*check_finite=*/true);
  if (a.rows == 0 || a.cols == 0) throw std::invalid_argument("matrix must be nonempty");
  if (std::sqrt(asq) == 0.0) throw std::invalid_argument("matrix must be nonzero");
  if (cfg.epsilon < 0.0) throw std::invalid_argument("epsilon must be nonnegative");
  if (cfg.b < 1) throw std::invalid_argument("block size must be at least 1");
  const Index min_dim = std::min(a.rows, a.cols);
  const Index max_rank = cfg.max_rank > 0 ? std::min<Index>(cfg.max_rank, min_dim) : min_dim;
  const Index max_iters = cfg.max_iters > 0 ? cfg.max_iters : (min_dim + cfg.b - 1) / cfg.b + 1;

  const auto run_start = Clock::now();
  auto t0 = Clock::now();
  SketchState st = make_sketch(cfg.seed, cfg.b, a, cfg.sketch_kind, cfg.sparse_nnz);
  res->sketch_s = seconds_since(t0);
  res->c = st.c;
  res->ga_norm = st.ga_norm;

  const double threshold =
      cfg.risk_adjust ? adjusted_threshold(cfg.epsilon, cfg.delta, cfg.alpha, st.c) : cfg.epsilon;
  res->threshold = threshold;

  double rho = downdate_col_residual(st, CurFactors{});
  if (rho <= threshold) {
    res->status = ORACLE_CONVERGED;
    res->final_rho = rho;
    std::snprintf(res->note, sizeof(res->note), "%s", "threshold at or above the initial estimate; empty factorization");
    res->total_s = seconds_since(run_start);
    return;
  }
  CurFactors cur;
  Index k = 0;
  int status = ORACLE_MAX_RANK;
  while (true) {
    if (cur.rank() >= max_rank || k >= max_iters) { status = ORACLE_MAX_RANK; break; }
    const auto it_start = Clock::now();
    const Index block = std::min(cfg.b, max_rank - cur.rank());
    SelectionResult colsel = select_columns(st.col_residual, block, cfg.col_method, cfg.pivot_floor, cur.J);
    if (colsel.indices.empty()) { status = ORACLE_RESIDUAL_EXHAUSTED; break; }
    log_steps(res, 0, k, colsel);
    const Mat s_row = row_residual(a, cur, colsel.indices);
    SelectionResult rowsel = select_rows(s_row, static_cast<Index>(colsel.indices.size()), cfg.row_method,
                                         cfg.pivot_floor, cur.I);
    if (rowsel.indices.empty()) { status = ORACLE_RESIDUAL_EXHAUSTED; break; }
    log_steps(res, 1, k, rowsel);
    const size_t width = std::min(colsel.indices.size(), rowsel.indices.size());
    IndexList nc = cur.J, nr = cur.I;
    nc.insert(nc.end(), colsel.indices.begin(), colsel.indices.begin() + static_cast<std::ptrdiff_t>(width));
    nr.insert(nr.end(), rowsel.indices.begin(), rowsel.indices.begin() + static_cast<std::ptrdiff_t>(width));
    CurFactors next;
    try {
      next = make_cur_factors(a, std::move(nr), std::move(nc));
    } catch (const std::runtime_error&) {
      status = ORACLE_RESIDUAL_EXHAUSTED;
      break;
    }
    cur = std::move(next);
    rho = downdate_col_residual(st, cur);
    if (k < res->cap_iters) {
      if (res->cod_rank) res->cod_rank[k] = cur.core.cod.rank;
      res->rhos[k] = rho;
      res->widths[k] = static_cast<Index>(width);
      if (res->iter_seconds) res->iter_seconds[k] = seconds_since(it_start);
    }
    ++k;
    if (rho <= threshold) { status = ORACLE_CONVERGED; break; }
  }
  res->n_iters = k;
  res->rank = cur.rank();
  for (Index q = 0; q < cur.rank() && q < res->cap_rank; ++q) {
    res->row_indices[q] = cur.I[static_cast<size_t>(q)];
    res->col_indices[q] = cur.J[static_cast<size_t>(q)];
  }
  res->status = status;
  res->final_rho = rho;
  res->total_s = seconds_since(run_start);
}

// true_relative_error, driver.cpp:169-190
double true_relative_error(const View& a, const CurFactors& cur) {
  double asq = 0.0;
  for (Index j = 0; j < a.cols; ++j) asq += sq_norm(a.p + j * a.ld, a.rows);
  const double a_norm = std::sqrt(asq);
  if (a_norm == 0.0) return 0.0;
  if (cur.empty()) return 1.0;
  constexpr Index kPanel = 256;
  double sq = 0.0;
  for (Index start = 0; start < a.cols; start += kPanel) {
    const Index stop = std::min(start + kPanel, a.cols);
    IndexList panel;
    for (Index j = start; j < stop; ++j) panel.push_back(j);
    Mat diff = gather_cols(a, panel);
    const Mat core_r = apply_pinv_left(cur.core, gather_cols(view(cur.R), panel));
    gemm_acc(cur.C, core_r, diff, -1.0);
    sq += sq_norm(diff.v.data(), static_cast<Index>(diff.v.size()));
  }
  return std::sqrt(sq) / a_norm;
}

}  // namespace oracle

// =====================================================================================
// C API
// =====================================================================================
namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
  try {
    f();
    return ORACLE_OK;
  } catch (const std::out_of_range& e) {  // derives from logic_error: catch first
    g_err = e.what();
    return ORACLE_E_OUT_OF_RANGE;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return ORACLE_E_DOMAIN;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORACLE_E_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return ORACLE_E_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORACLE_E_RUNTIME;
  }
}
oracle::IndexList to_list(const int64_t* p, int64_t n) { return oracle::IndexList(p, p + (n > 0 ? n : 0)); }
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }
int oracle_set_threads(int n) {
  oracle::g_thread_limit.store(n < 1 ? (1 << 30) : n);
  return oracle::Pool::get().size();
}

void oracle_philox4x32(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  const auto r = oracle::philox({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int k = 0; k < 4; ++k) out[k] = r[k];
}
double oracle_normal_at(uint64_t seed, uint32_t stream, int64_t i, int64_t j) {
  return oracle::normal_at(seed, stream, i, j);
}
double oracle_uniform_at(uint64_t seed, uint32_t stream, int64_t i, int64_t j) {
  return oracle::uniform_at(seed, stream, i, j);
}
void oracle_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, uint32_t stream, double* out) {
  oracle::parallel_for(0, cols, rows * cols > 65536, [&](int64_t j) {
    for (int64_t i = 0; i < rows; ++i) out[i + j * rows] = oracle::normal_at(seed, stream, i, j);
  });
}
void oracle_gaussian_fill(int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint32_t stream, double scale,
                          double* out) {
  oracle::parallel_for(0, cols, rows * cols > 65536, [&](int64_t j) {
    for (int64_t i = 0; i < rows; ++i) out[i + j * ld] = scale * oracle::normal_at(seed, stream, i, j);
  });
}
int oracle_sparse_sign_pattern(int64_t c, int64_t m, uint64_t seed, int32_t zeta, int32_t* rows_out,
                               int8_t* signs_out) {
  return guarded([&] {
    if (c < 1 || zeta < 1) throw std::invalid_argument("sparse-sign needs c >= 1 and zeta >= 1");
    const int ze = static_cast<int>(std::min<int64_t>(zeta, c));
    for (int64_t i = 0; i < m; ++i) oracle::sparse_sign_column(seed, i, c, ze, rows_out + i * ze, signs_out + i * ze);
  });
}
int64_t oracle_sketch_rows_for_block(int64_t b) { return oracle::sketch_rows_for_block(b); }
int oracle_sketch(const double* A, int64_t m, int64_t n, int64_t lda, int64_t b, uint64_t seed, int32_t kind,
                  int32_t zeta, double* Y, double* ga_norm, double* a_norm) {
  return guarded([&] {
    const oracle::View a{A, m, n, lda};
    oracle::SketchState st = oracle::make_sketch(seed, b, a, kind, zeta);
    std::memcpy(Y, st.sketched_input.v.data(), sizeof(double) * st.sketched_input.v.size());
    if (ga_norm) *ga_norm = st.ga_norm;
    if (a_norm) *a_norm = st.a_norm;
  });
}
int oracle_select(const double* M, int64_t rows, int64_t cols, int64_t ldm, int64_t b, int32_t is_columns,
                  int32_t method, double pivot_floor, const int64_t* exclude, int64_t n_exclude, int64_t* idx_out,
                  int64_t* n_idx, int32_t* truncated, double* last_pivot, double* best_out, double* second_out) {
  return guarded([&] {
    oracle::Mat m(rows, cols);
    for (int64_t j = 0; j < cols; ++j)
      for (int64_t i = 0; i < rows; ++i) m(i, j) = M[i + j * ldm];
    const auto ex = to_list(exclude, n_exclude);
    const auto r = is_columns ? oracle::select_columns(m, b, method, pivot_floor, ex)
                              : oracle::select_rows(m, b, method, pivot_floor, ex);
    *n_idx = static_cast<int64_t>(r.indices.size());
    for (size_t k = 0; k < r.indices.size(); ++k) {
      idx_out[k] = r.indices[k];
      if (best_out) best_out[k] = r.best[k];
      if (second_out) second_out[k] = r.second[k];
    }
    *truncated = r.truncated ? 1 : 0;
    *last_pivot = r.last_pivot_magnitude;
  });
}
int oracle_adjusted_threshold(double epsilon, double delta, double alpha, int64_t c, double* out) {
  return guarded([&] { *out = oracle::adjusted_threshold(epsilon, delta, alpha, c); });
}
int oracle_gratton_tail(int64_t c, double tau, double* out) {
  return guarded([&] { *out = oracle::gratton_tail(c, tau); });
}
int oracle_iterative_cur(const double* A, int64_t m, int64_t n, int64_t lda, const oracle_config* cfg,
                         oracle_result* res) {
  return guarded([&] {
    res->rank = res->n_iters = res->n_steps = 0;
    res->status = ORACLE_CONVERGED;
    res->final_rho = 1.0;
    res->threshold = res->sketch_s = res->total_s = res->ga_norm = 0.0;
    res->c = 0;
    res->note[0] = '\0';
    const int method_ok = (cfg->col_method >= 0 && cfg->col_method <= 2 && cfg->row_method >= 0 && cfg->row_method <= 2);
    if (!method_ok) throw std::invalid_argument("unknown selection method");
    oracle::iterative_cur(oracle::View{A, m, n, lda}, *cfg, res);
  });
}
int oracle_true_relative_error(const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I,
                               const int64_t* J, int64_t r, double* out) {
  return guarded([&] {
    const oracle::View a{A, m, n, lda};
    oracle::CurFactors cur;
    if (r > 0) cur = oracle::make_cur_factors(a, to_list(I, r), to_list(J, r));
    *out = oracle::true_relative_error(a, cur);
  });
}
int oracle_core_matrix(const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I, const int64_t* J,
                       int64_t r, double* core_out) {
  return guarded([&] {
    const oracle::View a{A, m, n, lda};
    oracle::CurFactors cur = oracle::make_cur_factors(a, to_list(I, r), to_list(J, r));
    oracle::Mat eye(r, r);
    for (int64_t i = 0; i < r; ++i) eye(i, i) = 1.0;
    const oracle::Mat p = cur.core.cod.solve(eye);  // FactoredPinv::materialize, pinv.cpp:40-43
    std::memcpy(core_out, p.v.data(), sizeof(double) * p.v.size());
  });
}

int oracle_core_solve(const double* A, int64_t m, int64_t n, int64_t lda, const int64_t* I, const int64_t* J,
                      int64_t r, const double* rhs, int64_t k, int64_t ldrhs, double* out) {
  return guarded([&] {
    const oracle::View a{A, m, n, lda};
    const auto Il = to_list(I, r), Jl = to_list(J, r);
    oracle::check_distinct(Il, "row");
    oracle::check_distinct(Jl, "column");
    oracle::Mat cross(r, r);  // gather_block, matrix.cpp:224-227
    for (int64_t q = 0; q < r; ++q)
      for (int64_t p = 0; p < r; ++p) {
        if (Il[p] < 0 || Il[p] >= m) oracle::bad_index("gather_rows", Il[p], m);
        if (Jl[q] < 0 || Jl[q] >= n) oracle::bad_index("gather_cols", Jl[q], n);
        cross(p, q) = a(Il[p], Jl[q]);
      }
    const oracle::FactoredPinv core = oracle::build_pinv(cross);
    oracle::Mat b(r, k);
    for (int64_t j = 0; j < k; ++j) std::memcpy(b.col(j), rhs + j * ldrhs, sizeof(double) * r);
    const oracle::Mat x = oracle::apply_pinv_left(core, b);
    std::memcpy(out, x.v.data(), sizeof(double) * x.v.size());
  });
}

// slupp_cur, proj/src/baselines.cpp:39-62: one sketch of ceil(1.1 r) rows (stream
// SluppSketch), r LUPP column pivots, LUPP row pivots on A(:, J), then the factors.
int oracle_slupp_cur(const double* A, int64_t m, int64_t n, int64_t lda, int64_t r, uint64_t seed, int64_t* I,
                     int64_t* J, int64_t* rank) {
  return guarded([&] {
    const oracle::View a{A, m, n, lda};
    if (r < 0 || r > std::min(m, n)) throw std::invalid_argument("rank must lie in [0, min(m, n)]");
    *rank = 0;
    if (r == 0) return;
    const int64_t c = (11 * r + 9) / 10;  // ceil(1.1 r)
    const oracle::Mat g = oracle::gaussian_matrix(c, m, seed, ORACLE_STREAM_SLUPP_SKETCH);
    oracle::Mat sketched(c, n);  // matmul(G, A)
    for (int64_t j = 0; j < n; ++j) {
      double* y = sketched.col(j);
      const double* aj = A + j * lda;
      for (int64_t k = 0; k < m; ++k) {
        const double* gk = g.col(k);
        for (int64_t i = 0; i < c; ++i) y[i] += gk[i] * aj[k];
      }
    }
    const oracle::SelectionResult cols =
        oracle::select_columns(sketched, std::min(r, c), ORACLE_PIVOT_LUPP, 1e-13, {});
    if (cols.indices.empty()) throw std::runtime_error("singular cross block");
    const oracle::Mat picked = oracle::gather_cols(a, cols.indices);
    const oracle::SelectionResult rows = oracle::select_rows(picked, static_cast<int64_t>(cols.indices.size()),
                                                             ORACLE_PIVOT_LUPP, 1e-13, {});
    if (rows.indices.empty()) throw std::runtime_error("singular cross block");
    const size_t width = std::min(cols.indices.size(), rows.indices.size());
    oracle::IndexList Ik(rows.indices.begin(), rows.indices.begin() + static_cast<std::ptrdiff_t>(width));
    oracle::IndexList Jk(cols.indices.begin(), cols.indices.begin() + static_cast<std::ptrdiff_t>(width));
    const oracle::CurFactors cur = oracle::make_cur_factors(a, Ik, Jk);  // may throw "singular cross block"
    for (size_t q = 0; q < width; ++q) {
      I[q] = cur.I[q];
      J[q] = cur.J[q];
    }
    *rank = static_cast<int64_t>(width);
  });
}

// Reference test fixtures (proj/tests/oracles.hpp:20-37): std::mt19937_64 with libstdc++'s
// uniform_real_distribution / normal_distribution, filled column by column — the exact
// inputs the reference's own unit tests use (g++/libstdc++ here, as there).
void oracle_fixture_random_dense(int64_t rows, int64_t cols, uint32_t seed, double lo, double hi, double* out) {
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) out[i + j * rows] = dist(gen);
}
void oracle_fixture_random_gaussian(int64_t rows, int64_t cols, uint32_t seed, double* out) {
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> dist;
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) out[i + j * rows] = dist(gen);
}

}  // extern "C"

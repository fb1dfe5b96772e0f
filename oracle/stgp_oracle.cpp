// stgp CPU oracle: restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY (see stgp_oracle.h).  Every function cites the
// reference file:line it restates; paths are relative to /root/reference/proj.
// Built with -ffp-contract=off (the reference's Release build has no -march, so
// its user code contains no contracted FMAs, proj/CMakeLists.txt:6-8).
#include "stgp_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <dlfcn.h>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct DataError : std::runtime_error {
  explicit DataError(const std::string& m) : std::runtime_error(m) {}
};
struct NumericError : std::runtime_error {
  explicit NumericError(const std::string& m) : std::runtime_error(m) {}
};

thread_local std::string g_err;
bool g_prune = true;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

constexpr double kLog2Pi = 1.8378770664093453;  // approximations.cpp:24

// types.hpp:65-70
inline uint64_t mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Pt {
  double x, y, t;
};

// types.hpp:53-57
inline double sdist(const Pt& a, const Pt& b) {
  const double dx = a.x - b.x, dy = a.y - b.y;
  return std::sqrt(dx * dx + dy * dy);
}
inline double tlag(const Pt& a, const Pt& b) { return std::abs(a.t - b.t); }

// covariance.cpp:34-46
void validate(const orc_params& p) {
  auto fail = [](const char* w) { throw ConfigError(std::string("CovarianceParams: ") + w); };
  if (!(p.sigma2 >= 0.0) || !std::isfinite(p.sigma2)) fail("sigma2 must be >= 0");
  if (!(p.sigma1_2 > 0.0) || !std::isfinite(p.sigma1_2)) fail("sigma1_2 must be > 0");
  if (!(p.a > 0.0) || !std::isfinite(p.a)) fail("a must be > 0");
  if (!(p.c > 0.0) || !std::isfinite(p.c)) fail("c must be > 0");
  if (!(p.alpha > 0.0 && p.alpha <= 1.0)) fail("alpha must be in (0, 1]");
  if (!(p.nu > 0.0) || !std::isfinite(p.nu)) fail("nu must be > 0");
  if (!(p.beta >= 0.0 && p.beta <= 1.0)) fail("beta must be in [0, 1]");
  if (!(p.delta >= 0.0) || !std::isfinite(p.delta)) fail("delta must be >= 0");
}

bool closed_form(double nu) { return nu == 0.5 || nu == 1.5 || nu == 2.5; }

// covariance.cpp:66-77
double matern(double x, double nu) {
  if (x < 0.0) throw ConfigError("matern_corr: x must be >= 0");
  if (x == 0.0) return 1.0;
  if (nu == 0.5) return std::exp(-x);
  if (nu == 1.5) return (1.0 + x) * std::exp(-x);
  if (nu == 2.5) return (1.0 + x + x * x / 3.0) * std::exp(-x);
  const double v = std::pow(2.0, 1.0 - nu) / std::tgamma(nu) * std::pow(x, nu) *
                   std::cyl_bessel_k(nu, x);
  return std::isfinite(v) ? v : 0.0;
}

// covariance.cpp:79-87
double matern_d(double x, double nu) {
  if (x < 0.0) throw ConfigError("matern_corr_deriv: x must be >= 0");
  if (nu == 0.5) return -std::exp(-x);
  if (nu == 1.5) return -x * std::exp(-x);
  if (nu == 2.5) return -(x * (1.0 + x) / 3.0) * std::exp(-x);
  throw NumericError("matern_corr_deriv: analytic derivative only for nu in {0.5, 1.5, 2.5}");
}

struct Temporal {
  double pow_mE, pow_mbh, inv_T, log_T, u2a, u2a_logu;
};

// GneitingKernel (covariance.cpp:89-181), including the integer-lag table and
// its 1e-9 snap rule (covariance.cpp:115-146).
struct Kernel {
  orc_params th{};
  double E = 0.0;
  std::vector<Temporal> table;

  explicit Kernel(const orc_params& p) : th(p) {
    validate(th);
    E = th.delta + th.beta * 2 / 2.0;
  }

  Temporal live(double u) const {
    Temporal f;
    if (u == 0.0) {
      f = {1.0, 1.0, 1.0, 0.0, 0.0, 0.0};
      return f;
    }
    f.u2a = std::pow(u, 2.0 * th.alpha);
    f.u2a_logu = f.u2a * std::log(u);
    const double T = th.a * f.u2a + 1.0;
    f.inv_T = 1.0 / T;
    f.log_T = std::log(T);
    f.pow_mE = std::pow(T, -E);
    f.pow_mbh = std::pow(T, -th.beta / 2.0);
    return f;
  }

  void precompute(int max_lag) {
    if (max_lag < 0 || max_lag > 2000000) throw ConfigError("GneitingKernel: unreasonable time-lag table size");
    table.resize(static_cast<size_t>(max_lag) + 1);
    for (int u = 0; u <= max_lag; ++u) table[static_cast<size_t>(u)] = live(static_cast<double>(u));
  }

  Temporal factors(double u) const {
    if (!table.empty()) {
      const double r = std::nearbyint(u);
      if (std::abs(u - r) < 1e-9 && r >= 0.0) {
        const int lag = static_cast<int>(r);
        if (lag < static_cast<int>(table.size())) return table[static_cast<size_t>(lag)];
      }
    }
    return live(u);
  }

  double eval(double h, double u) const {
    const Temporal f = factors(u);
    const double x = th.c * h * f.pow_mbh;
    return th.sigma1_2 * f.pow_mE * matern(x, th.nu);
  }
  double operator()(const Pt& a, const Pt& b) const { return eval(sdist(a, b), tlag(a, b)); }

  void grad(double h, double u, double g[6]) const {
    if (!closed_form(th.nu)) throw NumericError("GneitingKernel::grad: analytic gradient requires nu in {0.5, 1.5, 2.5}");
    const Temporal f = factors(u);
    const double x = th.c * h * f.pow_mbh;
    const double M = matern(x, th.nu);
    const double Mp = matern_d(x, th.nu);
    const double base = th.sigma1_2 * f.pow_mE;
    g[0] = f.pow_mE * M;
    const double dC_dT = base * f.inv_T * (-E * M - 0.5 * th.beta * x * Mp);
    g[1] = dC_dT * f.u2a;
    g[3] = dC_dT * 2.0 * th.a * f.u2a_logu;
    g[2] = base * Mp * x / th.c;
    g[4] = -f.log_T * base * (M + 0.5 * x * Mp);
    g[5] = -f.log_T * base * M;
  }
  void grad(const Pt& a, const Pt& b, double g[6]) const { grad(sdist(a, b), tlag(a, b), g); }
};

// approximations.cpp:26-38
void maybe_precompute_lags(Kernel& k, const std::vector<Pt>& pts) {
  double tmin = pts[0].t, tmax = pts[0].t;
  for (const auto& p : pts) {
    const double r = std::nearbyint(p.t);
    if (std::abs(p.t - r) >= 1e-9) return;
    tmin = std::min(tmin, p.t);
    tmax = std::max(tmax, p.t);
  }
  const double range = tmax - tmin;
  if (range >= 0.0 && range <= 200000.0) k.precompute(static_cast<int>(range) + 1);
}

// ---------------------------------------------------------------------------
// dense helpers (column-major); every accumulation is a sequential fma chain
// ---------------------------------------------------------------------------
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int r_, int c_) : r(r_), c(c_), a(static_cast<size_t>(r_) * c_, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(i) + static_cast<size_t>(j) * r]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(i) + static_cast<size_t>(j) * r]; }
  double* col(int j) { return a.data() + static_cast<size_t>(j) * r; }
  const double* col(int j) const { return a.data() + static_cast<size_t>(j) * r; }
};

inline double dot_seq(const double* a, const double* b, int n) {
  double acc = 0.0;
  for (int k = 0; k < n; ++k) acc = std::fma(a[k], b[k], acc);
  return acc;
}

// ---------------------------------------------------------------------------
// Optional BLAS timing mode (orc_set_blas): the dense n x M^2 contractions -- W = L^{-1} U, the Woodbury
// cores, the gradient's triangular solves and Gram products -- go to an OpenBLAS (the scipy-bundled one,
// LP64 Fortran symbols) the way the reference hands them to Eigen's blocked GEMM/TRSM
// (approximations.cpp:269-306, 513-536, 595-601, 711).  Results then differ from the sequential-order
// restatement by rounding only (~1e-13 relative); parity checks keep the default sequential order, the
// CPU baseline of bench.py uses this mode.
// ---------------------------------------------------------------------------
using dgemm_fn = void (*)(const char*, const char*, const int*, const int*, const int*, const double*, const double*,
                          const int*, const double*, const int*, const double*, double*, const int*);
using dsyrk_fn = void (*)(const char*, const char*, const int*, const int*, const double*, const double*, const int*,
                          const double*, double*, const int*);
using dtrsm_fn = void (*)(const char*, const char*, const char*, const char*, const int*, const int*, const double*,
                          const double*, const int*, double*, const int*);
struct Blas {
  dgemm_fn gemm = nullptr;
  dsyrk_fn syrk = nullptr;
  dtrsm_fn trsm = nullptr;
  void (*set_threads)(int) = nullptr;
};
Blas g_blas_fns;
bool g_blas = false;

// C (r x c) = alpha op(A) op(B) + beta C, all column-major Mats
void blas_gemm(bool ta, bool tb, double alpha, const Mat& A, const Mat& B, double beta, Mat& C) {
  const int m = C.r, n = C.c, k = ta ? A.r : A.c;
  const int lda = std::max(1, A.r), ldb = std::max(1, B.r), ldc = std::max(1, C.r);
  if (m == 0 || n == 0) return;
  g_blas_fns.gemm(ta ? "T" : "N", tb ? "T" : "N", &m, &n, &k, &alpha, A.a.data(), &lda, B.a.data(), &ldb, &beta,
                  C.a.data(), &ldc);
}
// C (lower) = alpha A A^T + beta C, A n x k
void blas_syrk(double alpha, const Mat& A, double beta, Mat& C) {
  const int n = A.r, k = A.c, lda = std::max(1, A.r), ldc = std::max(1, C.r);
  if (n == 0) return;
  g_blas_fns.syrk("L", "N", &n, &k, &alpha, A.a.data(), &lda, &beta, C.a.data(), &ldc);
}

// Cholesky A = L L^T, lower triangle, row-major scratch Lr (n*n) for speed.
// Fails when a pivot is <= 0 (Eigen's LLT info() != Success criterion).
// Element (r,c) accumulates A(r,c) - sum_{k<c} L(r,k) L(c,k) in increasing k.
bool chol_seq(const Mat& A, Mat& L) {
  const int n = A.r;
  L = Mat(n, n);
  std::vector<double> Lr(static_cast<size_t>(n) * n, 0.0);  // row-major lower
  for (int j = 0; j < n; ++j) {
    double acc = A(j, j);
    const double* Lj = &Lr[static_cast<size_t>(j) * n];
    for (int k = 0; k < j; ++k) acc = std::fma(-Lj[k], Lj[k], acc);
    if (!(acc > 0.0)) {
      if (acc <= 0.0) return false;
    }
    const double d = std::sqrt(acc);
    Lr[static_cast<size_t>(j) * n + j] = d;
#pragma omp parallel for schedule(static) if (n - j > 256)
    for (int r = j + 1; r < n; ++r) {
      double s = A(r, j);
      const double* Lrr = &Lr[static_cast<size_t>(r) * n];
      for (int k = 0; k < j; ++k) s = std::fma(-Lrr[k], Lj[k], s);
      Lr[static_cast<size_t>(r) * n + j] = s / d;
    }
  }
  for (int r = 0; r < n; ++r)
    for (int c = 0; c <= r; ++c) L(r, c) = Lr[static_cast<size_t>(r) * n + c];
  return true;
}

// L x = b, forward substitution, x[r] = (b[r] - sum_{c<r} L(r,c) x[c]) / L(r,r)
// with the sum as a sequential fma chain.  Lrow is row-major lower.
void fwd_seq(const std::vector<double>& Lrow, int n, const double* b, double* x) {
  for (int r = 0; r < n; ++r) {
    double acc = b[r];
    const double* Lr = &Lrow[static_cast<size_t>(r) * n];
    for (int c = 0; c < r; ++c) acc = std::fma(-Lr[c], x[c], acc);
    x[r] = acc / Lr[r];
  }
}
// L^T x = y (back substitution)
void bwd_seq(const std::vector<double>& Lrow, int n, const double* y, double* x) {
  for (int r = n - 1; r >= 0; --r) {
    double acc = y[r];
    for (int c = r + 1; c < n; ++c) acc = std::fma(-Lrow[static_cast<size_t>(c) * n + r], x[c], acc);
    x[r] = acc / Lrow[static_cast<size_t>(r) * n + r];
  }
}
std::vector<double> rowmajor(const Mat& L) {
  std::vector<double> o(static_cast<size_t>(L.r) * L.r);
  for (int r = 0; r < L.r; ++r)
    for (int c = 0; c <= r; ++c) o[static_cast<size_t>(r) * L.r + c] = L(r, c);
  return o;
}

struct Chol {
  int n = 0;
  std::vector<double> Lr;  // row-major lower
  bool ok = false;
  bool compute(const Mat& A) {
    Mat L;
    ok = chol_seq(A, L);
    n = A.r;
    if (ok) Lr = rowmajor(L);
    return ok;
  }
  void solve(const double* b, double* x) const {
    std::vector<double> y(static_cast<size_t>(n));
    fwd_seq(Lr, n, b, y.data());
    bwd_seq(Lr, n, y.data(), x);
  }
  void lsolve(const double* b, double* x) const { fwd_seq(Lr, n, b, x); }
  double logdet() const {  // 2 sum log diag
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += std::log(Lr[static_cast<size_t>(i) * n + i]);
    return 2.0 * s;
  }
  double diag(int i) const { return Lr[static_cast<size_t>(i) * n + i]; }
  // B <- L^{-1} B (trans: L^{-T} B) through BLAS, B n x ncols column-major
  void trsm(Mat& B, bool trans) const {
    if (Lc.empty()) {
      auto& self = const_cast<Chol&>(*this);
      self.Lc.assign(static_cast<size_t>(n) * n, 0.0);
      for (int r = 0; r < n; ++r)
        for (int c = 0; c <= r; ++c) self.Lc[static_cast<size_t>(c) * n + r] = Lr[static_cast<size_t>(r) * n + c];
    }
    const int m = B.r, nc = B.c, ld = std::max(1, n), ldb = std::max(1, B.r);
    const double one = 1.0;
    if (m == 0 || nc == 0) return;
    g_blas_fns.trsm("L", "L", trans ? "T" : "N", "N", &m, &nc, &one, Lc.data(), &ld, B.a.data(), &ldb);
  }
  std::vector<double> Lc;  // column-major copy of L for BLAS (lazily formed)
};

// Mc (lower, symmetrized) += sum_i A(:,i) A(:,i)^T / d_i through BLAS (scaled copy + SYRK)
void blas_core(const Mat& A, const std::vector<double>& d, Mat& Mc) {
  Mat As = A;
  for (int i = 0; i < A.c; ++i) {
    const double sc = 1.0 / std::sqrt(d[static_cast<size_t>(i)]);
    for (int j = 0; j < A.r; ++j) As(j, i) *= sc;
  }
  blas_syrk(1.0, As, 1.0, Mc);
  for (int a = 0; a < Mc.r; ++a)
    for (int b = 0; b < a; ++b) Mc(b, a) = Mc(a, b);
}

// ---------------------------------------------------------------------------
// InducingBasis (inducing.cpp:237-284)
// ---------------------------------------------------------------------------
struct Basis {
  std::vector<Pt> z;
  Mat sigma;  // jittered
  Chol llt;
  int m() const { return static_cast<int>(z.size()); }
  Basis() = default;
  Basis(const std::vector<Pt>& pts, const Kernel& k) : z(pts) {
    const int M = m();
    if (M == 0) return;
    sigma = Mat(M, M);
    for (int i = 0; i < M; ++i)
      for (int j = 0; j <= i; ++j) {
        const double v = k(z[static_cast<size_t>(i)], z[static_cast<size_t>(j)]);
        sigma(i, j) = v;
        sigma(j, i) = v;
      }
    const double jitter = 1e-8 * k.th.sigma1_2;
    Mat jit = sigma;
    for (int i = 0; i < M; ++i) jit(i, i) += jitter;
    if (!llt.compute(jit)) {
      for (int i = 0; i < M; ++i) jit(i, i) += 9.0 * jitter;
      if (!llt.compute(jit)) throw NumericError("InducingBasis: inducing covariance is not positive definite");
    }
    sigma = jit;
  }
  // whitened cross covariance w = L^{-1} k_m(p), k_m(p)[j] = k(z_j, p)
  void whiten_point(const Kernel& k, const Pt& p, double* kvec, double* w) const {
    const int M = m();
    for (int j = 0; j < M; ++j) kvec[j] = k(z[static_cast<size_t>(j)], p);
    fwd_seq(llt.Lr, M, kvec, w);
  }
};

// U (M x n) and W = L^{-1} U (M x n)
// exact = true keeps the sequential fma chain even in BLAS mode: the searches' d_r distances are defined
// by it bit for bit
void cross_and_whiten(const Basis& b, const Kernel& k, const std::vector<Pt>& pts, Mat* U, Mat& W,
                      bool exact = false) {
  const int M = b.m(), n = static_cast<int>(pts.size());
  W = Mat(M, n);
  if (U) *U = Mat(M, n);
  if (g_blas && !exact) {  // U by kernel evaluations, then one TRSM
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < M; ++j) W(j, i) = k(b.z[static_cast<size_t>(j)], pts[static_cast<size_t>(i)]);
    if (U) *U = W;
    b.llt.trsm(W, false);
    return;
  }
#pragma omp parallel
  {
    std::vector<double> kv(static_cast<size_t>(M));
#pragma omp for schedule(static)
    for (int i = 0; i < n; ++i) {
      b.whiten_point(k, pts[static_cast<size_t>(i)], kv.data(), W.col(i));
      if (U) std::copy(kv.begin(), kv.end(), U->col(i));
    }
  }
}

std::vector<Pt> make_pts(int n, const double* x, const double* y, const double* t) {
  std::vector<Pt> p(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    if (!std::isfinite(x[i]) || !std::isfinite(y[i]) || !std::isfinite(t[i]))
      throw DataError("SpaceTimePoint: coordinates and time must be finite");
    p[static_cast<size_t>(i)] = {x[i], y[i], t[i]};
  }
  return p;
}

// ---------------------------------------------------------------------------
// neighbour searches
// ---------------------------------------------------------------------------
// neighbors.cpp:37-43 (DcMetric)
inline double dc_metric(const Kernel& k, const Pt& a, const Pt& b) {
  const double rho = k(a, b) / k.th.sigma1_2;
  return std::sqrt(std::max(1.0 - std::abs(rho), 0.0));
}

// brute_force_knn (tests/oracles.cpp:157-168) == cover-tree kNN
// (neighbors.cpp:150-226, proven equal by test_neighbors.cpp:96-131).
// `dist(j)` returns metric(i, j).  Rows are ascending, -1 padded.
template <class DistFn>
void topm_scan(int i, int m_v, DistFn&& dist, const std::vector<std::pair<int, int>>* blocks,
               const std::vector<double>* block_lb2, int32_t* out, double* dout) {
  const int want = std::min(m_v, i);
  for (int k = 0; k < m_v; ++k) {
    out[k] = -1;
    if (dout) dout[k] = std::numeric_limits<double>::quiet_NaN();
  }
  if (want <= 0) return;
  // max-heap of (d, j) lexicographic
  std::vector<std::pair<double, int>> heap;
  heap.reserve(static_cast<size_t>(want) + 1);
  auto consider = [&](int j) {
    const double d = dist(j);
    const std::pair<double, int> c{d, j};
    if (static_cast<int>(heap.size()) < want) {
      heap.push_back(c);
      std::push_heap(heap.begin(), heap.end());
    } else if (c < heap.front()) {
      std::pop_heap(heap.begin(), heap.end());
      heap.back() = c;
      std::push_heap(heap.begin(), heap.end());
    }
  };
  if (blocks == nullptr) {
    for (int j = 0; j < i; ++j) consider(j);
  } else {
    // blocks: [start, end) of equal time, ascending; scan backwards from i
    for (int b = static_cast<int>(blocks->size()) - 1; b >= 0; --b) {
      const int s = (*blocks)[static_cast<size_t>(b)].first;
      const int e = std::min((*blocks)[static_cast<size_t>(b)].second, i);
      if (s >= e) continue;
      if (static_cast<int>(heap.size()) == want) {
        const double dm = heap.front().first;
        if ((*block_lb2)[static_cast<size_t>(b)] - 1e-12 > dm * dm) continue;  // exact prune
      }
      for (int j = e - 1; j >= s; --j) consider(j);
    }
  }
  std::sort(heap.begin(), heap.end());
  std::vector<int> idx;
  for (const auto& h : heap) idx.push_back(h.second);
  if (dout)
    for (size_t k = 0; k < heap.size(); ++k) dout[k] = heap[k].first;  // by distance
  std::sort(idx.begin(), idx.end());
  for (size_t k = 0; k < idx.size(); ++k) out[k] = idx[k];
}

bool time_sorted(const std::vector<Pt>& p) {
  for (size_t i = 1; i < p.size(); ++i)
    if (p[i].t < p[i - 1].t) return false;
  return true;
}
std::vector<std::pair<int, int>> time_blocks(const std::vector<Pt>& p) {
  std::vector<std::pair<int, int>> b;
  int s = 0;
  for (int i = 1; i <= static_cast<int>(p.size()); ++i)
    if (i == static_cast<int>(p.size()) || p[static_cast<size_t>(i)].t != p[static_cast<size_t>(s)].t) {
      b.emplace_back(s, i);
      s = i;
    }
  return b;
}

// ---------------------------------------------------------------------------
// kMeans++ (inducing.cpp:22-115)
// ---------------------------------------------------------------------------
int count_distinct_rows(const Mat& P) {
  std::set<std::vector<double>> seen;
  for (int i = 0; i < P.r; ++i) {
    std::vector<double> row(static_cast<size_t>(P.c));
    for (int j = 0; j < P.c; ++j) row[static_cast<size_t>(j)] = P(i, j);
    seen.insert(std::move(row));
  }
  return static_cast<int>(seen.size());
}

// Eigen's VectorXd::sum() for a contiguous, 16-byte aligned vector on SSE2:
// two Packet2d accumulators striding 4, combined, one tail packet, lane0+lane1,
// scalar tail (Eigen Redux.h LinearVectorizedTraversal; Eigen is not vendored,
// so this is the oracle's definition).
double eigen_sum(const double* w, long n) {
  if (n <= 0) return 0.0;
  const long aligned = (n / 2) * 2;
  if (aligned == 0) {
    double r = w[0];
    for (long i = 1; i < n; ++i) r += w[i];
    return r;
  }
  const long aligned2 = (n / 4) * 4;
  double p0a = w[0], p0b = w[1];
  if (aligned > 2) {
    double p1a = w[2], p1b = w[3];
    for (long i = 4; i < aligned2; i += 4) {
      p0a += w[i];
      p0b += w[i + 1];
      p1a += w[i + 2];
      p1b += w[i + 3];
    }
    p0a += p1a;
    p0b += p1b;
    if (aligned > aligned2) {
      p0a += w[aligned2];
      p0b += w[aligned2 + 1];
    }
  }
  double r = p0a + p0b;
  for (long i = aligned; i < n; ++i) r += w[i];
  return r;
}

inline double row_sqnorm_diff(const Mat& P, int i, const Mat& C, int j) {
  double r = 0.0;
  for (int c = 0; c < P.c; ++c) {
    const double d = P(i, c) - C(j, c);
    r = (c == 0) ? d * d : r + d * d;
  }
  return r;
}

long weighted_pick(const std::vector<double>& w, std::mt19937_64& rng) {
  const double total = eigen_sum(w.data(), static_cast<long>(w.size()));
  std::uniform_real_distribution<double> unif(0.0, total);
  const double u = unif(rng);
  double acc = 0.0;
  for (size_t i = 0; i < w.size(); ++i) {
    acc += w[i];
    if (u <= acc) return static_cast<long>(i);
  }
  return static_cast<long>(w.size()) - 1;
}

Mat kmeanspp(const Mat& P, int k, uint64_t seed) {
  const int n = P.r;
  if (n == 0) throw DataError("kmeanspp: no points");
  if (k < 1) throw ConfigError("kmeanspp: k must be >= 1");
  if (k > count_distinct_rows(P)) throw DataError("kmeanspp: k exceeds the number of distinct points");
  std::mt19937_64 rng(mix_seed(seed, 0x6d70));
  Mat C(k, P.c);
  std::uniform_int_distribution<long> first(0, n - 1);
  const long f = first(rng);
  for (int c = 0; c < P.c; ++c) C(0, c) = P(static_cast<int>(f), c);
  std::vector<double> d2(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) d2[static_cast<size_t>(i)] = row_sqnorm_diff(P, i, C, 0);
  for (int j = 1; j < k; ++j) {
    const long pick = weighted_pick(d2, rng);
    for (int c = 0; c < P.c; ++c) C(j, c) = P(static_cast<int>(pick), c);
    for (int i = 0; i < n; ++i) {
      const double v = row_sqnorm_diff(P, i, C, j);
      d2[static_cast<size_t>(i)] = std::min(d2[static_cast<size_t>(i)], v);
    }
  }
  std::vector<int> assign(static_cast<size_t>(n), -1);
  double prev = std::numeric_limits<double>::infinity();
  for (int sweep = 0; sweep < 50; ++sweep) {
    double inertia = 0.0;
    for (int i = 0; i < n; ++i) {
      double best = std::numeric_limits<double>::infinity();
      int bj = 0;
      for (int j = 0; j < k; ++j) {
        const double d = row_sqnorm_diff(P, i, C, j);
        if (d < best) {
          best = d;
          bj = j;
        }
      }
      assign[static_cast<size_t>(i)] = bj;
      inertia += best;
    }
    Mat sums(k, P.c);
    std::vector<int> counts(static_cast<size_t>(k), 0);
    for (int i = 0; i < n; ++i) {
      const int a = assign[static_cast<size_t>(i)];
      for (int c = 0; c < P.c; ++c) sums(a, c) += P(i, c);
      ++counts[static_cast<size_t>(a)];
    }
    for (int j = 0; j < k; ++j) {
      if (counts[static_cast<size_t>(j)] > 0) {
        for (int c = 0; c < P.c; ++c) C(j, c) = sums(j, c) / counts[static_cast<size_t>(j)];
      } else {
        int far = 0;
        double fd = -1.0;
        for (int i = 0; i < n; ++i) {
          const double d = row_sqnorm_diff(P, i, C, assign[static_cast<size_t>(i)]);
          if (d > fd) {
            fd = d;
            far = i;
          }
        }
        for (int c = 0; c < P.c; ++c) C(j, c) = P(far, c);
      }
    }
    if (inertia == 0.0 || std::abs(prev - inertia) < 1e-6 * std::max(inertia, 1e-300)) break;
    prev = inertia;
  }
  return C;
}

// ---------------------------------------------------------------------------
// Vecchia rows (approximations.cpp:42-152)
// ---------------------------------------------------------------------------
struct Nbrs {
  int n = 0, m_v = 0;
  const int32_t* idx = nullptr;
  int count(int i) const {
    int c = 0;
    const int32_t* r = idx + static_cast<size_t>(i) * m_v;
    while (c < m_v && r[c] >= 0) ++c;
    return c;
  }
  const int32_t* row(int i) const { return idx + static_cast<size_t>(i) * m_v; }
};

struct BlockCov {
  const std::vector<Pt>* pts;
  const Kernel* k;
  double nugget;
  const Mat* W;  // whitened, may be null / empty
  double operator()(int a, int b) const {
    double v = (*k)((*pts)[static_cast<size_t>(a)], (*pts)[static_cast<size_t>(b)]);
    if (W && W->r > 0) v -= dot_seq(W->col(a), W->col(b), W->r);
    if (a == b) v += nugget;
    return v;
  }
};

struct RowFactors {
  int k = 0;
  std::vector<double> A, c;
  double D = 0.0;
  Chol llt;
};

// solve_row (approximations.cpp:69-111) with the jitter ladder
RowFactors solve_row(const BlockCov& cov, const int32_t* N, int k, int i, double s1) {
  RowFactors o;
  o.k = k;
  o.c.resize(static_cast<size_t>(k));
  Mat C(k, k);
  for (int a = 0; a < k; ++a) {
    o.c[static_cast<size_t>(a)] = cov(i, N[a]);
    for (int b = 0; b <= a; ++b) {
      const double v = cov(N[a], N[b]);
      C(a, b) = v;
      C(b, a) = v;
    }
  }
  const double dii = cov(i, i);
  if (k == 0) {
    o.D = dii;
    if (!(o.D > 0.0)) throw NumericError("vecchia row: non-positive marginal variance");
    return o;
  }
  if (!o.llt.compute(C)) {
    double jitter = 1e-10 * s1;
    for (int attempt = 0; attempt < 2; ++attempt) {
      for (int a = 0; a < k; ++a) C(a, a) += jitter;
      if (o.llt.compute(C)) break;
      jitter *= 9.0;
    }
    if (!o.llt.ok) throw NumericError("vecchia row: conditioning block is not positive definite");
  }
  o.A.resize(static_cast<size_t>(k));
  o.llt.solve(o.c.data(), o.A.data());
  double ac = 0.0;
  for (int a = 0; a < k; ++a) ac += o.A[static_cast<size_t>(a)] * o.c[static_cast<size_t>(a)];
  o.D = dii - ac;
  if (!(o.D > 0.0)) throw NumericError("vecchia row: non-positive conditional variance (near-duplicate points)");
  return o;
}

struct Rows {
  std::vector<double> D;
  std::vector<double> A;  // n * m_v, aligned with neighbour ELL
};

Rows assemble(const std::vector<Pt>& pts, const BlockCov& cov, const Nbrs& nb, double s1) {
  const int n = static_cast<int>(pts.size());
  if (nb.n != n) throw ConfigError("build: neighbor sets inconsistent with the dataset");
  Rows r;
  r.D.assign(static_cast<size_t>(n), 0.0);
  r.A.assign(static_cast<size_t>(n) * nb.m_v, 0.0);
  std::string err;
  int code = 0;
#pragma omp parallel for schedule(dynamic, 32)
  for (int i = 0; i < n; ++i) {
    try {
      RowFactors rf = solve_row(cov, nb.row(i), nb.count(i), i, s1);
      r.D[static_cast<size_t>(i)] = rf.D;
      for (int a = 0; a < rf.k; ++a) r.A[static_cast<size_t>(i) * nb.m_v + a] = rf.A[static_cast<size_t>(a)];
    } catch (const NumericError& e) {
#pragma omp critical
      if (!code) {
        code = 4;
        err = e.what();
      }
    } catch (const std::exception& e) {
#pragma omp critical
      if (!code) {
        code = 1;
        err = e.what();
      }
    }
  }
  if (code == 4) throw NumericError(err);
  if (code) throw std::runtime_error(err);
  return r;
}

// sparse products with B (unit lower, -A on N(i)), approximations.cpp:154-173
void b_apply(const Nbrs& nb, const Rows& R, const double* v, double* out) {
  const int n = nb.n;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    const int k = nb.count(i);
    const int32_t* N = nb.row(i);
    double acc = 0.0;
    for (int a = 0; a < k; ++a) acc += -R.A[static_cast<size_t>(i) * nb.m_v + a] * v[N[a]];
    acc += 1.0 * v[i];
    out[i] = acc;
  }
}
void bt_apply(const Nbrs& nb, const Rows& R, const double* v, double* out) {
  const int n = nb.n;
  std::fill(out, out + n, 0.0);
  for (int i = 0; i < n; ++i) {
    const int k = nb.count(i);
    const int32_t* N = nb.row(i);
    for (int a = 0; a < k; ++a) out[N[a]] += -R.A[static_cast<size_t>(i) * nb.m_v + a] * v[i];
    out[i] += v[i];
  }
}
std::vector<double> q_apply(const Nbrs& nb, const Rows& R, const double* v) {
  const int n = nb.n;
  std::vector<double> u(static_cast<size_t>(n)), o(static_cast<size_t>(n));
  b_apply(nb, R, v, u.data());
  for (int i = 0; i < n; ++i) u[static_cast<size_t>(i)] /= R.D[static_cast<size_t>(i)];
  bt_apply(nb, R, u.data(), o.data());
  return o;
}
// Sigma_s v = B^{-1} D B^{-T} v
std::vector<double> sigma_s_apply(const Nbrs& nb, const Rows& R, const double* v) {
  const int n = nb.n;
  std::vector<double> x(v, v + n);
  // B^T x' = x (unit upper): backward
  for (int i = n - 1; i >= 0; --i) {
    const int k = nb.count(i);
    const int32_t* N = nb.row(i);
    for (int a = 0; a < k; ++a) x[static_cast<size_t>(N[a])] -= -R.A[static_cast<size_t>(i) * nb.m_v + a] * x[static_cast<size_t>(i)];
  }
  for (int i = 0; i < n; ++i) x[static_cast<size_t>(i)] *= R.D[static_cast<size_t>(i)];
  // B x'' = x (unit lower): forward
  for (int i = 0; i < n; ++i) {
    const int k = nb.count(i);
    const int32_t* N = nb.row(i);
    double acc = x[static_cast<size_t>(i)];
    for (int a = 0; a < k; ++a) acc -= -R.A[static_cast<size_t>(i) * nb.m_v + a] * x[static_cast<size_t>(N[a])];
    x[static_cast<size_t>(i)] = acc;
  }
  return x;
}

std::vector<double> residual(int n, const double* yv, int p, const double* X, const double* beta) {
  std::vector<double> r(yv, yv + n);
  if (p > 0 && beta) {
    for (int i = 0; i < n; ++i) {
      double xb = 0.0;
      for (int j = 0; j < p; ++j) xb += X[static_cast<size_t>(i) + static_cast<size_t>(j) * n] * beta[j];
      r[static_cast<size_t>(i)] -= xb;
    }
  }
  return r;
}

// ---------------------------------------------------------------------------
// model assembly shared by all entry points
// ---------------------------------------------------------------------------
struct Model {
  int kind = 0, policy = 0, n = 0;
  std::vector<Pt> pts;
  Nbrs nb;
  Kernel kernel;
  Basis basis;
  Mat U, W;   // M x n
  Rows rows;  // Vecchia / VIF residual factors
  // FITC
  std::vector<double> fitc_diag, lambda;
  Chol Mllt;  // Woodbury core (FITC / VIF)
  Model(const orc_model* m) : kernel(m->theta) {}
};

void build_model(Model& s, const orc_model* m) {
  validate(m->theta);
  s.kind = m->kind;
  s.policy = m->policy;
  s.n = m->n;
  if (s.n < 1) throw DataError("SpaceTimeDataset: empty dataset");
  s.pts = make_pts(m->n, m->x, m->y, m->t);
  maybe_precompute_lags(s.kernel, s.pts);
  s.nb.n = m->n;
  s.nb.m_v = m->m_v;
  s.nb.idx = m->nbr;
  const double s1 = m->theta.sigma1_2;
  std::vector<Pt> z;
  if (m->kind != 0)
    for (int j = 0; j < m->M; ++j) z.push_back({m->zx[j], m->zy[j], m->zt[j]});
  if (m->kind == 0) {  // build_vecchia, approximations.cpp:198-213
    const double nug = m->policy == 1 ? m->theta.sigma2 : 0.0;
    BlockCov cov{&s.pts, &s.kernel, nug, nullptr};
    s.rows = assemble(s.pts, cov, s.nb, s1);
    return;
  }
  if (m->kind == 1) {  // build_fitc, approximations.cpp:238-275
    if (m->M < 1) throw ConfigError("build_fitc: need at least one inducing point");
    s.basis = Basis(z, s.kernel);
    cross_and_whiten(s.basis, s.kernel, s.pts, &s.U, s.W);
    const int n = s.n, M = s.basis.m();
    s.fitc_diag.resize(static_cast<size_t>(n));
    const double clamp_tol = 1e-10 * std::max(1.0, s1);
    for (int i = 0; i < n; ++i) {
      double d = s1 - dot_seq(s.W.col(i), s.W.col(i), M);
      if (d < 0.0) {
        if (d < -clamp_tol) throw NumericError("build_fitc: diagonal correction went negative");
        d = 0.0;
      }
      s.fitc_diag[static_cast<size_t>(i)] = d;
    }
    s.lambda.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      s.lambda[static_cast<size_t>(i)] = s.fitc_diag[static_cast<size_t>(i)] + m->theta.sigma2;
      if (s.lambda[static_cast<size_t>(i)] <= 0.0)
        throw NumericError("build_fitc: zero observation diagonal; a positive nugget is required");
    }
    Mat Mc = s.basis.sigma;
    if (g_blas) {
      blas_core(s.U, s.lambda, Mc);
    } else {
#pragma omp parallel for schedule(dynamic)
      for (int a = 0; a < M; ++a)
        for (int b = 0; b <= a; ++b) {
          double acc = 0.0;
          for (int i = 0; i < n; ++i) acc += s.U(a, i) * s.U(b, i) / s.lambda[static_cast<size_t>(i)];
          Mc(a, b) += acc;
          if (a != b) Mc(b, a) = Mc(a, b);
        }
    }
    if (!s.Mllt.compute(Mc)) throw NumericError("build_fitc: Woodbury core factorization failed");
    return;
  }
  // build_vif, approximations.cpp:277-312
  s.basis = Basis(z, s.kernel);
  const int M = s.basis.m(), n = s.n;
  if (M > 0) {
    cross_and_whiten(s.basis, s.kernel, s.pts, &s.U, s.W);
  } else {
    s.W = Mat(0, n);
    s.U = Mat(0, n);
  }
  const double nug = m->policy == 1 ? m->theta.sigma2 : 0.0;
  BlockCov cov{&s.pts, &s.kernel, nug, &s.W};
  s.rows = assemble(s.pts, cov, s.nb, s1);
  if (M > 0) {
    // M = Sigma_m + U Q U^T = Sigma_m + VB D^{-1} VB^T with VB = U B^T
    Mat VB(M, n);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      const int k = s.nb.count(i);
      const int32_t* N = s.nb.row(i);
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int a = 0; a < k; ++a) acc += -s.rows.A[static_cast<size_t>(i) * s.nb.m_v + a] * s.U(j, N[a]);
        acc += s.U(j, i);
        VB(j, i) = acc;
      }
    }
    Mat Mc = s.basis.sigma;
    if (g_blas) {
      blas_core(VB, s.rows.D, Mc);
    } else {
#pragma omp parallel for schedule(dynamic)
      for (int a = 0; a < M; ++a)
        for (int b = 0; b <= a; ++b) {
          double acc = 0.0;
          for (int i = 0; i < n; ++i) acc += VB(a, i) * VB(b, i) / s.rows.D[static_cast<size_t>(i)];
          Mc(a, b) += acc;
          if (a != b) Mc(b, a) = Mc(a, b);
        }
    }
    if (!s.Mllt.compute(Mc)) throw NumericError("build_vif: Woodbury core factorization failed");
  }
}

void require_obs(const Model& s, const char* what) {
  if (s.kind != 1 && s.policy != 1)
    throw NumericError(std::string(what) + ": requires the observation-policy structure");
}

// nll (approximations.cpp:336-384); latent policy goes through the Laplace
// algebra, which is out of scope
double nll_model(const Model& s, const std::vector<double>& r) {
  const int n = s.n;
  if (s.kind == 0) {
    if (s.policy != 1) throw ConfigError("nll: latent-policy likelihood needs the Laplace algebra (out of scope)");
    std::vector<double> u(static_cast<size_t>(n));
    b_apply(s.nb, s.rows, r.data(), u.data());
    double acc = 0.0;
    for (int i = 0; i < n; ++i) {
      const double D = s.rows.D[static_cast<size_t>(i)];
      acc += std::log(D) + u[static_cast<size_t>(i)] * u[static_cast<size_t>(i)] / D;
    }
    return 0.5 * (acc + n * kLog2Pi);
  }
  const int M = s.basis.m();
  if (s.kind == 1) {
    std::vector<double> rl(static_cast<size_t>(n)), v(static_cast<size_t>(M)), Mv(static_cast<size_t>(M));
    for (int i = 0; i < n; ++i) rl[static_cast<size_t>(i)] = r[static_cast<size_t>(i)] / s.lambda[static_cast<size_t>(i)];
    for (int j = 0; j < M; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += s.U(j, i) * rl[static_cast<size_t>(i)];
      v[static_cast<size_t>(j)] = acc;
    }
    s.Mllt.solve(v.data(), Mv.data());
    double quad = 0.0;
    for (int i = 0; i < n; ++i) quad += r[static_cast<size_t>(i)] * rl[static_cast<size_t>(i)];
    double vMv = 0.0;
    for (int j = 0; j < M; ++j) vMv += v[static_cast<size_t>(j)] * Mv[static_cast<size_t>(j)];
    quad -= vMv;
    double logdet = 0.0;
    for (int i = 0; i < n; ++i) logdet += std::log(s.lambda[static_cast<size_t>(i)]);
    logdet -= s.basis.llt.logdet();
    logdet += s.Mllt.logdet();
    return 0.5 * (logdet + quad + n * kLog2Pi);
  }
  if (s.policy != 1) throw ConfigError("nll: latent-policy likelihood needs the Laplace algebra (out of scope)");
  const std::vector<double> ur = q_apply(s.nb, s.rows, r.data());
  double logdet = 0.0;
  for (int i = 0; i < n; ++i) logdet += std::log(s.rows.D[static_cast<size_t>(i)]);
  double quad = 0.0;
  for (int i = 0; i < n; ++i) quad += r[static_cast<size_t>(i)] * ur[static_cast<size_t>(i)];
  if (M > 0) {
    std::vector<double> w(static_cast<size_t>(M)), Mw(static_cast<size_t>(M));
    for (int j = 0; j < M; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += s.U(j, i) * ur[static_cast<size_t>(i)];
      w[static_cast<size_t>(j)] = acc;
    }
    s.Mllt.solve(w.data(), Mw.data());
    double wMw = 0.0;
    for (int j = 0; j < M; ++j) wMw += w[static_cast<size_t>(j)] * Mw[static_cast<size_t>(j)];
    quad -= wMw;
    logdet += s.Mllt.logdet() - s.basis.llt.logdet();
  }
  return 0.5 * (logdet + quad + n * kLog2Pi);
}

inline void add_pair(const Kernel& k, const Pt& a, const Pt& b, double w, double* g) {
  double kg[6];
  k.grad(a, b, kg);
  for (int q = 0; q < 6; ++q) g[q + 1] += w * kg[q];
}

// nll_grad Vecchia (approximations.cpp:403-493)
// scale (nullable): per component, the sum over rows of |row contribution| -- the conditioning of the
// gradient sum, the yardstick of the parity tolerance
void grad_vecchia(const Model& s, const std::vector<double>& r, double* grad, double* scale) {
  if (s.policy != 1) throw NumericError("nll_grad: analytic gradient is defined for the observation-policy structure driven by the optimizer");
  const int n = s.n;
  const orc_params& th = s.kernel.th;
  std::vector<double> u(static_cast<size_t>(n));
  b_apply(s.nb, s.rows, r.data(), u.data());
  BlockCov cov{&s.pts, &s.kernel, th.sigma2, nullptr};
  std::vector<double> part(static_cast<size_t>(n) * 7, 0.0);
  int code = 0;
  std::string err;
  double g00[6];
  s.kernel.grad(0.0, 0.0, g00);
#pragma omp parallel for schedule(dynamic, 32)
  for (int i = 0; i < n; ++i) {
    try {
      const int k = s.nb.count(i);
      const int32_t* N = s.nb.row(i);
      RowFactors rf = solve_row(cov, N, k, i, th.sigma1_2);
      std::vector<double> w(static_cast<size_t>(k));
      for (int a = 0; a < k; ++a) w[static_cast<size_t>(a)] = r[static_cast<size_t>(N[a])];
      if (k > 0) {
        std::vector<double> tmp(w);
        rf.llt.solve(tmp.data(), w.data());
      }
      double An = 0.0, Aw = 0.0;
      for (int a = 0; a < k; ++a) {
        An += rf.A[static_cast<size_t>(a)] * rf.A[static_cast<size_t>(a)];
        Aw += rf.A[static_cast<size_t>(a)] * w[static_cast<size_t>(a)];
      }
      const double s1n = 1.0 + (k > 0 ? An : 0.0);
      const double s2n = k > 0 ? -Aw : 0.0;
      double s1[6] = {0}, s2[6] = {0};
      for (int a = 0; a < k; ++a) {
        const Pt& pa = s.pts[static_cast<size_t>(N[a])];
        const double ta = -rf.A[static_cast<size_t>(a)];
        const double wa = w[static_cast<size_t>(a)];
        double kg[6];
        s.kernel.grad(pa, s.pts[static_cast<size_t>(i)], kg);
        for (int q = 0; q < 6; ++q) {
          s1[q] += 2.0 * ta * kg[q];
          s2[q] += wa * kg[q];
        }
        for (int b = 0; b < a; ++b) {
          const Pt& pb = s.pts[static_cast<size_t>(N[b])];
          s.kernel.grad(pa, pb, kg);
          const double tb = -rf.A[static_cast<size_t>(b)];
          const double wb = w[static_cast<size_t>(b)];
          for (int q = 0; q < 6; ++q) {
            s1[q] += 2.0 * ta * tb * kg[q];
            s2[q] += (wa * tb + wb * ta) * kg[q];
          }
        }
        for (int q = 0; q < 6; ++q) {
          s1[q] += ta * ta * g00[q];
          s2[q] += wa * ta * g00[q];
        }
      }
      for (int q = 0; q < 6; ++q) s1[q] += g00[q];
      const double Di = rf.D;
      const double ui = u[static_cast<size_t>(i)];
      const double cd = 0.5 * (1.0 / Di - ui * ui / (Di * Di));
      const double cu = ui / Di;
      double* g = &part[static_cast<size_t>(i) * 7];
      g[0] = cd * s1n - cu * s2n;
      for (int q = 0; q < 6; ++q) g[q + 1] = cd * s1[q] - cu * s2[q];
    } catch (const NumericError& e) {
#pragma omp critical
      if (!code) {
        code = 4;
        err = e.what();
      }
    }
  }
  if (code) throw NumericError(err);
  for (int q = 0; q < 7; ++q) grad[q] = 0.0;
  for (int i = 0; i < n; ++i)
    for (int q = 0; q < 7; ++q) grad[q] += part[static_cast<size_t>(i) * 7 + q];
  if (scale) {
    for (int q = 0; q < 7; ++q) scale[q] = 0.0;
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < 7; ++q) scale[q] += std::abs(part[static_cast<size_t>(i) * 7 + q]);
  }
}

// U-pair and Sigma_m-pair kernel-gradient sums shared by FITC and VIF: sum_{j,i} om(j,i) dk(z_j, p_i) and
// sum_{j1,j2} wsig(j1,j2) dk(z_j1, z_j2); each data column i and each inducing row j1 is one contribution
// to the scale.
template <class Om>
void lowrank_pairs(const Model& s, int M, Om&& om, const Mat& wsig, double* grad, double* scale) {
  const int n = s.n;
  const int T = std::max(1, omp_get_max_threads());
  std::vector<double> loc(static_cast<size_t>(T) * 14, 0.0);
#pragma omp parallel
  {
    double* g = &loc[static_cast<size_t>(omp_get_thread_num()) * 14];
#pragma omp for schedule(static)
    for (int i = 0; i < n; ++i) {
      double gi[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int j = 0; j < M; ++j) add_pair(s.kernel, s.basis.z[static_cast<size_t>(j)], s.pts[static_cast<size_t>(i)], om(j, i), gi);
      for (int q = 0; q < 7; ++q) {
        g[q] += gi[q];
        g[7 + q] += std::abs(gi[q]);
      }
    }
  }
  for (int tt = 0; tt < T; ++tt)
    for (int q = 0; q < 7; ++q) {
      grad[q] += loc[static_cast<size_t>(tt) * 14 + q];
      if (scale) scale[q] += loc[static_cast<size_t>(tt) * 14 + 7 + q];
    }
  for (int j1 = 0; j1 < M; ++j1) {
    double gj[7] = {0, 0, 0, 0, 0, 0, 0};
    add_pair(s.kernel, s.basis.z[static_cast<size_t>(j1)], s.basis.z[static_cast<size_t>(j1)], wsig(j1, j1), gj);
    for (int j2 = 0; j2 < j1; ++j2)
      add_pair(s.kernel, s.basis.z[static_cast<size_t>(j1)], s.basis.z[static_cast<size_t>(j2)], wsig(j1, j2) + wsig(j2, j1), gj);
    for (int q = 0; q < 7; ++q) {
      grad[q] += gj[q];
      if (scale) scale[q] += std::abs(gj[q]);
    }
  }
}

// helper: Y = Cholesky-solve of each column (M x n)
Mat chol_solve_cols(const Chol& c, const Mat& B) {
  if (g_blas) {
    Mat X = B;
    c.trsm(X, false);
    c.trsm(X, true);
    return X;
  }
  Mat X(B.r, B.c);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < B.c; ++i) c.solve(B.col(i), X.col(i));
  return X;
}
Mat chol_lsolve_cols(const Chol& c, const Mat& B) {
  if (g_blas) {
    Mat X = B;
    c.trsm(X, false);
    return X;
  }
  Mat X(B.r, B.c);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < B.c; ++i) c.lsolve(B.col(i), X.col(i));
  return X;
}

// nll_grad FITC (approximations.cpp:495-571)
void grad_fitc(const Model& s, const std::vector<double>& r, double* grad, double* scale) {
  const int n = s.n, M = s.basis.m();
  const Mat& U = s.U;
  std::vector<double> lam_inv(static_cast<size_t>(n)), rl(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    lam_inv[static_cast<size_t>(i)] = 1.0 / s.lambda[static_cast<size_t>(i)];
    rl[static_cast<size_t>(i)] = r[static_cast<size_t>(i)] * lam_inv[static_cast<size_t>(i)];
  }
  std::vector<double> v(static_cast<size_t>(M)), Mv(static_cast<size_t>(M)), alpha(static_cast<size_t>(n));
  for (int j = 0; j < M; ++j) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += U(j, i) * rl[static_cast<size_t>(i)];
    v[static_cast<size_t>(j)] = acc;
  }
  s.Mllt.solve(v.data(), Mv.data());
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int j = 0; j < M; ++j) acc += U(j, i) * Mv[static_cast<size_t>(j)];
    alpha[static_cast<size_t>(i)] = rl[static_cast<size_t>(i)] - lam_inv[static_cast<size_t>(i)] * acc;
  }
  const Mat P = chol_solve_cols(s.basis.llt, U);
  Mat UL(M, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < M; ++j) UL(j, i) = U(j, i) * lam_inv[static_cast<size_t>(i)];
  const Mat H = chol_lsolve_cols(s.Mllt, UL);
  std::vector<double> dsinv(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    double sq = 0.0;
    for (int j = 0; j < M; ++j) sq += H(j, i) * H(j, i);
    dsinv[static_cast<size_t>(i)] = lam_inv[static_cast<size_t>(i)] - sq / 1.0;
  }
  const Mat NL = chol_solve_cols(s.Mllt, UL);
  Mat G1(M, M);  // P * UL^T
  Mat K2(M, n);
  Mat W2(M, M);  // K2 P^T
  if (g_blas) {
    blas_gemm(false, true, 1.0, P, UL, 0.0, G1);
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < M; ++a) K2(a, i) = P(a, i) * lam_inv[static_cast<size_t>(i)];
    blas_gemm(false, false, -1.0, G1, NL, 1.0, K2);
    blas_gemm(false, true, 1.0, K2, P, 0.0, W2);
  } else {
#pragma omp parallel for schedule(static)
    for (int a = 0; a < M; ++a)
      for (int b = 0; b < M; ++b) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += P(a, i) * UL(b, i);
        G1(a, b) = acc;
      }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < M; ++a) {
        double acc = 0.0;
        for (int b = 0; b < M; ++b) acc += G1(a, b) * NL(b, i);
        K2(a, i) = P(a, i) * lam_inv[static_cast<size_t>(i)] - acc;
      }
#pragma omp parallel for schedule(static)
    for (int a = 0; a < M; ++a)
      for (int b = 0; b < M; ++b) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += K2(a, i) * P(b, i);
        W2(a, b) = acc;
      }
  }
  std::vector<double> Pa(static_cast<size_t>(M)), phi(static_cast<size_t>(n));
  for (int a = 0; a < M; ++a) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += P(a, i) * alpha[static_cast<size_t>(i)];
    Pa[static_cast<size_t>(a)] = acc;
  }
  for (int i = 0; i < n; ++i)
    phi[static_cast<size_t>(i)] = 0.5 * (dsinv[static_cast<size_t>(i)] - alpha[static_cast<size_t>(i)] * alpha[static_cast<size_t>(i)]);
  Mat wsig(M, M);
  if (g_blas) {
    Mat Pphi = P;
    for (int i = 0; i < n; ++i)
      for (int a = 0; a < M; ++a) Pphi(a, i) *= phi[static_cast<size_t>(i)];
    blas_gemm(false, true, 1.0, Pphi, P, 0.0, wsig);
    for (int a = 0; a < M; ++a)
      for (int b = 0; b < M; ++b)
        wsig(a, b) += -0.5 * W2(a, b) + 0.5 * (Pa[static_cast<size_t>(a)] * Pa[static_cast<size_t>(b)]);
  } else {
#pragma omp parallel for schedule(static)
    for (int a = 0; a < M; ++a)
      for (int b = 0; b < M; ++b) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += P(a, i) * phi[static_cast<size_t>(i)] * P(b, i);
        wsig(a, b) = -0.5 * W2(a, b) + 0.5 * (Pa[static_cast<size_t>(a)] * Pa[static_cast<size_t>(b)]) + acc;
      }
  }
  for (int q = 0; q < 7; ++q) grad[q] = 0.0;
  if (scale)
    for (int q = 0; q < 7; ++q) scale[q] = 0.0;
  double phisum = 0.0, phiabs = 0.0;
  for (int i = 0; i < n; ++i) {
    phisum += phi[static_cast<size_t>(i)];
    phiabs += std::abs(phi[static_cast<size_t>(i)]);
  }
  grad[0] += phisum;
  grad[1] += phisum;
  if (scale) {
    scale[0] += phiabs;
    scale[1] += phiabs;
  }
  auto om = [&](int j, int i) {
    return K2(j, i) - Pa[static_cast<size_t>(j)] * alpha[static_cast<size_t>(i)] - P(j, i) * (2.0 * phi[static_cast<size_t>(i)]);
  };
  lowrank_pairs(s, M, om, wsig, grad, scale);
}

// nll_grad VIF (approximations.cpp:573-744).  Phi is kept as per-row dense
// (k+1)^2 blocks instead of one sparse n x n matrix; the direct pass and P*Phi
// then sum the same entries (the reference's lower-triangle + coeff(b,a) fold
// equals the full symmetric sum because d k is symmetric).
void grad_vif(const Model& s, const std::vector<double>& r, double* grad, double* scale) {
  require_obs(s, "nll_grad");
  const int n = s.n, M = s.basis.m();
  const orc_params& th = s.kernel.th;
  const Mat& U = s.U;
  BlockCov cov{&s.pts, &s.kernel, th.sigma2, &s.W};
  const std::vector<double> ur = q_apply(s.nb, s.rows, r.data());
  std::vector<double> t(static_cast<size_t>(n), 0.0), yM(static_cast<size_t>(M));
  Mat LVB, Hhat, N1;
  if (M > 0) {
    std::vector<double> w(static_cast<size_t>(M));
    for (int j = 0; j < M; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += U(j, i) * ur[static_cast<size_t>(i)];
      w[static_cast<size_t>(j)] = acc;
    }
    s.Mllt.solve(w.data(), yM.data());
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < M; ++j) acc += U(j, i) * yM[static_cast<size_t>(j)];
      t[static_cast<size_t>(i)] = acc;
    }
    Mat VB(M, n);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
      const int k = s.nb.count(i);
      const int32_t* N = s.nb.row(i);
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int a = 0; a < k; ++a) acc += U(j, N[a]) * -s.rows.A[static_cast<size_t>(i) * s.nb.m_v + a];
        acc += U(j, i);
        VB(j, i) = acc;
      }
    }
    LVB = chol_lsolve_cols(s.Mllt, VB);
    Hhat = Mat(M, n);
    if (g_blas) {
      Hhat = LVB;
      s.Mllt.trsm(Hhat, true);
    } else {
#pragma omp parallel for schedule(static)
      for (int i = 0; i < n; ++i) bwd_seq(s.Mllt.Lr, M, LVB.col(i), Hhat.col(i));
    }
    N1 = chol_solve_cols(s.Mllt, U);
  }
  std::vector<double> z(static_cast<size_t>(n)), Bz(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) z[static_cast<size_t>(i)] = r[static_cast<size_t>(i)] - t[static_cast<size_t>(i)];
  b_apply(s.nb, s.rows, z.data(), Bz.data());

  // per-row Phi blocks
  const int K1 = s.nb.m_v + 1;
  std::vector<double> phi(static_cast<size_t>(n) * K1 * K1, 0.0);
  int code = 0;
  std::string err;
#pragma omp parallel for schedule(dynamic, 32)
  for (int i = 0; i < n; ++i) {
    try {
      const int k = s.nb.count(i);
      const int32_t* N = s.nb.row(i);
      RowFactors rf = solve_row(cov, N, k, i, th.sigma1_2);
      const double Di = s.rows.D[static_cast<size_t>(i)];
      std::vector<double> at(static_cast<size_t>(k) + 1), Ga(static_cast<size_t>(k) + 1, 0.0),
          zcl(static_cast<size_t>(k) + 1), Rv(static_cast<size_t>(k) + 1, 0.0);
      for (int a = 0; a < k; ++a) at[static_cast<size_t>(a)] = -rf.A[static_cast<size_t>(a)];
      at[static_cast<size_t>(k)] = 1.0;
      double aGa = 0.0;
      if (M > 0) {
        const double* h = Hhat.col(i);
        for (int a = 0; a < k; ++a) {
          double acc = 0.0;
          for (int j = 0; j < M; ++j) acc += U(j, N[a]) * h[j];
          Ga[static_cast<size_t>(a)] = acc;
        }
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += U(j, i) * h[j];
        Ga[static_cast<size_t>(k)] = acc;
        double sq = 0.0;
        for (int j = 0; j < M; ++j) sq += LVB(j, i) * LVB(j, i);
        aGa = sq;
      }
      for (int a = 0; a < k; ++a) zcl[static_cast<size_t>(a)] = z[static_cast<size_t>(N[a])];
      zcl[static_cast<size_t>(k)] = z[static_cast<size_t>(i)];
      const double uz = Bz[static_cast<size_t>(i)];
      const double c0 = 0.5 * (1.0 / Di - (aGa + uz * uz) / (Di * Di));
      std::vector<double> vrow(static_cast<size_t>(k) + 1);
      for (int a = 0; a <= k; ++a) vrow[static_cast<size_t>(a)] = (Ga[static_cast<size_t>(a)] + uz * zcl[static_cast<size_t>(a)]) / Di;
      if (k > 0) rf.llt.solve(vrow.data(), Rv.data());
      Rv[static_cast<size_t>(k)] = 0.0;
      double* ph = &phi[static_cast<size_t>(i) * K1 * K1];
      for (int a = 0; a <= k; ++a)
        for (int b = 0; b <= k; ++b)
          ph[a * K1 + b] = c0 * at[static_cast<size_t>(a)] * at[static_cast<size_t>(b)] -
                           0.5 * (at[static_cast<size_t>(a)] * Rv[static_cast<size_t>(b)] + at[static_cast<size_t>(b)] * Rv[static_cast<size_t>(a)]);
    } catch (const NumericError& e) {
#pragma omp critical
      if (!code) {
        code = 4;
        err = e.what();
      }
    }
  }
  if (code) throw NumericError(err);
  auto clidx = [&](int i, int a) { return a < s.nb.count(i) ? s.nb.row(i)[a] : i; };

  for (int q = 0; q < 7; ++q) grad[q] = 0.0;
  {
    std::vector<double> part(static_cast<size_t>(n) * 7, 0.0);
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 0; i < n; ++i) {
      const int k = s.nb.count(i);
      const double* ph = &phi[static_cast<size_t>(i) * K1 * K1];
      double* g = &part[static_cast<size_t>(i) * 7];
      for (int a = 0; a <= k; ++a) {
        const int pa = clidx(i, a);
        add_pair(s.kernel, s.pts[static_cast<size_t>(pa)], s.pts[static_cast<size_t>(pa)], ph[a * K1 + a], g);
        g[0] += ph[a * K1 + a];
        for (int b = 0; b < a; ++b) {
          const int pb = clidx(i, b);
          add_pair(s.kernel, s.pts[static_cast<size_t>(pa)], s.pts[static_cast<size_t>(pb)], ph[a * K1 + b] + ph[b * K1 + a], g);
        }
      }
    }
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < 7; ++q) grad[q] += part[static_cast<size_t>(i) * 7 + q];
    if (scale) {
      for (int q = 0; q < 7; ++q) scale[q] = 0.0;
      for (int i = 0; i < n; ++i)
        for (int q = 0; q < 7; ++q) scale[q] += std::abs(part[static_cast<size_t>(i) * 7 + q]);
    }
  }
  if (M == 0) return;
  const Mat P = chol_solve_cols(s.basis.llt, U);
  // omega = (Q N1^T)^T - yM (ur - Q t)^T - 2 P Phi
  Mat omega(M, n);
#pragma omp parallel
  {
    std::vector<double> row(static_cast<size_t>(n));
#pragma omp for schedule(static)
    for (int j = 0; j < M; ++j) {
      for (int i = 0; i < n; ++i) row[static_cast<size_t>(i)] = N1(j, i);
      const std::vector<double> q = q_apply(s.nb, s.rows, row.data());
      for (int i = 0; i < n; ++i) omega(j, i) = q[static_cast<size_t>(i)];
    }
  }
  const std::vector<double> qt = q_apply(s.nb, s.rows, t.data());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < M; ++j) omega(j, i) -= yM[static_cast<size_t>(j)] * (ur[static_cast<size_t>(i)] - qt[static_cast<size_t>(i)]);
  // PPhi(j, pb) += sum_a P(j, pa) Phi_i(a, b), rows i in order, a in order; each thread owns a slice of
  // j so the column accesses stay contiguous (same per-element order as a j-outer loop)
  Mat PPhi(M, n);
#pragma omp parallel
  {
    const int T = omp_get_num_threads(), tid = omp_get_thread_num();
    const int j0 = static_cast<int>(static_cast<long>(M) * tid / T), j1 = static_cast<int>(static_cast<long>(M) * (tid + 1) / T);
    std::vector<double> acc(static_cast<size_t>(std::max(j1 - j0, 0)));
    for (int i = 0; i < n && j1 > j0; ++i) {
      const int k = s.nb.count(i);
      const double* ph = &phi[static_cast<size_t>(i) * K1 * K1];
      for (int b = 0; b <= k; ++b) {
        std::fill(acc.begin(), acc.end(), 0.0);
        for (int a = 0; a <= k; ++a) {
          const double w = ph[a * K1 + b];
          const double* Pa = P.col(clidx(i, a));
          for (int j = j0; j < j1; ++j) acc[static_cast<size_t>(j - j0)] += Pa[j] * w;
        }
        double* dst = PPhi.col(clidx(i, b));
        for (int j = j0; j < j1; ++j) dst[j] += acc[static_cast<size_t>(j - j0)];
      }
    }
  }
  for (size_t e = 0; e < omega.a.size(); ++e) omega.a[e] -= 2.0 * PPhi.a[e];
  // wsig = 0.5 yM yM^T + PPhi P^T + 0.5 (M^{-1} - Sigma_m^{-1})
  Mat wsig(M, M);
  if (g_blas) {
    blas_gemm(false, true, 1.0, PPhi, P, 0.0, wsig);
    for (int a = 0; a < M; ++a)
      for (int b = 0; b < M; ++b) wsig(a, b) += 0.5 * (yM[static_cast<size_t>(a)] * yM[static_cast<size_t>(b)]);
  } else {
#pragma omp parallel for schedule(static)
    for (int a = 0; a < M; ++a)
      for (int b = 0; b < M; ++b) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += PPhi(a, i) * P(b, i);
        wsig(a, b) = 0.5 * (yM[static_cast<size_t>(a)] * yM[static_cast<size_t>(b)]) + acc;
      }
  }
  {
    Mat I(M, M);
    for (int j = 0; j < M; ++j) I(j, j) = 1.0;
    const Mat Minv = chol_solve_cols(s.Mllt, I);
    const Mat Sinv = chol_solve_cols(s.basis.llt, I);
    for (size_t e = 0; e < wsig.a.size(); ++e) wsig.a[e] += 0.5 * (Minv.a[e] - Sinv.a[e]);
  }
  lowrank_pairs(s, M, [&](int j, int i) { return omega(j, i); }, wsig, grad, scale);
}

// gls_beta (approximations.cpp:752-798)
std::vector<double> sigma_inv_apply(const Model& s, const std::vector<double>& v) {
  const int n = s.n, M = s.basis.m();
  if (s.kind == 0) return q_apply(s.nb, s.rows, v.data());
  if (s.kind == 1) {
    std::vector<double> vl(static_cast<size_t>(n)), w(static_cast<size_t>(M)), Mw(static_cast<size_t>(M)), o(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) vl[static_cast<size_t>(i)] = v[static_cast<size_t>(i)] / s.lambda[static_cast<size_t>(i)];
    for (int j = 0; j < M; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += s.U(j, i) * vl[static_cast<size_t>(i)];
      w[static_cast<size_t>(j)] = acc;
    }
    s.Mllt.solve(w.data(), Mw.data());
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < M; ++j) acc += s.U(j, i) * Mw[static_cast<size_t>(j)];
      o[static_cast<size_t>(i)] = vl[static_cast<size_t>(i)] - acc / s.lambda[static_cast<size_t>(i)];
    }
    return o;
  }
  std::vector<double> qv = q_apply(s.nb, s.rows, v.data());
  if (M > 0) {
    std::vector<double> w(static_cast<size_t>(M)), Mw(static_cast<size_t>(M)), t(static_cast<size_t>(n));
    for (int j = 0; j < M; ++j) {
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += s.U(j, i) * qv[static_cast<size_t>(i)];
      w[static_cast<size_t>(j)] = acc;
    }
    s.Mllt.solve(w.data(), Mw.data());
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < M; ++j) acc += s.U(j, i) * Mw[static_cast<size_t>(j)];
      t[static_cast<size_t>(i)] = acc;
    }
    const std::vector<double> qt = q_apply(s.nb, s.rows, t.data());
    for (int i = 0; i < n; ++i) qv[static_cast<size_t>(i)] -= qt[static_cast<size_t>(i)];
  }
  return qv;
}

// symmetric positive definite p x p solve (LDLT in the reference)
std::vector<double> spd_solve(int p, std::vector<double> A, std::vector<double> b) {
  Mat Am(p, p);
  for (int i = 0; i < p * p; ++i) Am.a[static_cast<size_t>(i)] = A[static_cast<size_t>(i)];
  Chol c;
  if (!c.compute(Am)) throw NumericError("gls_beta: normal equations are singular");
  std::vector<double> x(static_cast<size_t>(p));
  c.solve(b.data(), x.data());
  return x;
}

// target_neighbors (approximations.cpp:816-863)
std::vector<int> target_nbrs(const Pt& q, const Model& s, int kind_metric, double ss, double ts,
                             const std::vector<double>* resid, const double* wq, double rq, int want_m) {
  const int n = s.n;
  const int want = std::min(want_m, n);
  std::vector<std::pair<double, int>> cand(static_cast<size_t>(n));
  const double s1 = s.kernel.th.sigma1_2;
  const int M = s.W.r;
  for (int j = 0; j < n; ++j) {
    double d;
    const Pt& pj = s.pts[static_cast<size_t>(j)];
    if (kind_metric == 0) {
      const double dx = (q.x - pj.x) / ss, dy = (q.y - pj.y) / ss, dt = (q.t - pj.t) / ts;
      d = dx * dx + dy * dy + dt * dt;
    } else if (kind_metric == 1) {
      d = 1.0 - std::abs(s.kernel(q, pj) / s1);
    } else {
      const double dj = (*resid)[static_cast<size_t>(j)];
      const double tol = 1e-7 * s1;
      if (dj <= tol || rq <= tol) {
        d = 1.0;
      } else {
        double rho = s.kernel(q, pj);
        if (M > 0) rho -= dot_seq(wq, s.W.col(j), M);
        d = 1.0 - std::abs(rho) / std::sqrt(dj * rq);
      }
    }
    cand[static_cast<size_t>(j)] = {d, j};
  }
  std::partial_sort(cand.begin(), cand.begin() + want, cand.end());
  std::vector<int> out(static_cast<size_t>(want));
  for (int k = 0; k < want; ++k) out[static_cast<size_t>(k)] = cand[static_cast<size_t>(k)].second;
  std::sort(out.begin(), out.end());
  return out;
}

}  // namespace

// ---------------------------------------------------------------------------
// Laplace algebra (approximations.cpp:1083-1375) and the ZC-PTN likelihood / Newton mode finding /
// prediction (laplace.cpp:25-259), dense at the oracle's sizes: the reference factors Q + W with a
// sparse LDLT (SimplicialLDLT), whose determinant and solves equal the dense Cholesky's up to rounding.
// ---------------------------------------------------------------------------
// Q = B^T D^{-1} B (form_precision, approximations.cpp:181-190)
Mat form_precision_dense(const Model& s) {
  const int n = s.n;
  Mat Q(n, n);
  for (int r = 0; r < n; ++r) {
    const int k = s.nb.count(r);
    const int32_t* N = s.nb.row(r);
    const double Dr = s.rows.D[static_cast<size_t>(r)];
    std::vector<int> idx(static_cast<size_t>(k) + 1);
    std::vector<double> val(static_cast<size_t>(k) + 1);
    for (int a = 0; a < k; ++a) {
      idx[static_cast<size_t>(a)] = N[a];
      val[static_cast<size_t>(a)] = -s.rows.A[static_cast<size_t>(r) * s.nb.m_v + a];
    }
    idx[static_cast<size_t>(k)] = r;
    val[static_cast<size_t>(k)] = 1.0;
    for (int a = 0; a <= k; ++a)
      for (int b = 0; b <= k; ++b)
        Q(idx[static_cast<size_t>(a)], idx[static_cast<size_t>(b)]) +=
            val[static_cast<size_t>(a)] * val[static_cast<size_t>(b)] / Dr;
  }
  return Q;
}

struct Laplace {
  const Model* s;
  int kind;
  // Vecchia / VIF: Q, the factor of S = Q + W and log|Sigma_s| = sum log D
  Mat Q;
  Chol S;
  double logdet_sigma = 0.0, logdet_S = 0.0;
  // VIF: QUt = Q U^T (n x M), Z = S^{-1} QUt, the core M_w
  Mat QUt, Z;
  Chol Mw;
  double logdet_Mw = 0.0;
  // FITC (approximations.cpp:1168-1200)
  std::vector<double> scale, e1;
  double logdet_fitc = 0.0;

  explicit Laplace(const Model& m) : s(&m), kind(m.kind) {
    if (kind != 1) {  // VecchiaLaplace / VifLaplace (approximations.cpp:1090-1097, 1230-1237)
      if (m.policy != 0) throw NumericError("LaplaceAlgebra: requires a latent-policy structure");
      Q = form_precision_dense(m);
      for (int i = 0; i < m.n; ++i) logdet_sigma += std::log(m.rows.D[static_cast<size_t>(i)]);
      const int M = m.basis.m();
      if (kind == 2 && M > 0) {  // QUt = sparse_q_apply(B, D, U^T) (approximations.cpp:303)
        QUt = Mat(m.n, M);
        std::vector<double> col(static_cast<size_t>(m.n));
        for (int j = 0; j < M; ++j) {
          for (int i = 0; i < m.n; ++i) col[static_cast<size_t>(i)] = m.U(j, i);
          const std::vector<double> q = q_apply(m.nb, m.rows, col.data());
          for (int i = 0; i < m.n; ++i) QUt(i, j) = q[static_cast<size_t>(i)];
        }
      }
    }
  }
  int n() const { return s->n; }
  // prepare(w) (approximations.cpp:1100-1108, 1168-1184, 1240-1259)
  void prepare(const std::vector<double>& w) {
    const int n_ = n(), M = s->basis.m();
    if (kind == 1) {
      const std::vector<double>& lam0 = s->fitc_diag;
      scale.assign(static_cast<size_t>(n_), 0.0);
      e1.assign(static_cast<size_t>(n_), 0.0);
      std::vector<double> dw(static_cast<size_t>(n_));
      for (int i = 0; i < n_; ++i) {
        scale[static_cast<size_t>(i)] = 1.0 / (1.0 + w[static_cast<size_t>(i)] * lam0[static_cast<size_t>(i)]);
        e1[static_cast<size_t>(i)] = lam0[static_cast<size_t>(i)] * scale[static_cast<size_t>(i)];
        dw[static_cast<size_t>(i)] = w[static_cast<size_t>(i)] * scale[static_cast<size_t>(i)];
      }
      Mat Mc = s->basis.sigma;
      for (int a = 0; a < M; ++a)
        for (int b = 0; b < M; ++b) {
          double acc = 0.0;
          for (int i = 0; i < n_; ++i) acc += s->U(a, i) * dw[static_cast<size_t>(i)] * s->U(b, i);
          Mc(a, b) += acc;
        }
      if (!Mw.compute(Mc)) throw NumericError("FitcLaplace: core factorization failed");
      double l1 = 0.0;
      for (int i = 0; i < n_; ++i) l1 += std::log(1.0 + w[static_cast<size_t>(i)] * lam0[static_cast<size_t>(i)]);
      logdet_fitc = l1 + Mw.logdet() - s->basis.llt.logdet();
      return;
    }
    Mat Sm = Q;
    for (int i = 0; i < n_; ++i) Sm(i, i) += w[static_cast<size_t>(i)];
    if (!S.compute(Sm)) throw NumericError(kind == 0 ? "VecchiaLaplace: factorization of Q + W failed"
                                                     : "VifLaplace: factorization of Q + W failed");
    logdet_S = S.logdet();
    if (kind == 2 && M > 0) {
      Z = chol_solve_cols(S, QUt);
      Mat Mc = s->basis.sigma;
      for (int a = 0; a < M; ++a)
        for (int b = 0; b < M; ++b) {
          double acc = 0.0, acc2 = 0.0;
          for (int i = 0; i < n_; ++i) {
            acc += s->U(a, i) * QUt(i, b);
            acc2 += QUt(i, a) * Z(i, b);
          }
          Mc(a, b) += acc - acc2;
        }
      for (int a = 0; a < M; ++a)  // symmetric by construction up to rounding: use the lower triangle
        for (int b = a + 1; b < M; ++b) Mc(a, b) = Mc(b, a);
      if (!Mw.compute(Mc)) throw NumericError("VifLaplace: core factorization failed");
      logdet_Mw = Mw.logdet();
    }
  }
  // (Sigma^{-1} + W)^{-1} x
  std::vector<double> solve(const std::vector<double>& x) const {
    const int n_ = n(), M = s->basis.m();
    std::vector<double> out(static_cast<size_t>(n_));
    if (kind == 1) {
      std::vector<double> tx(static_cast<size_t>(M)), mt(static_cast<size_t>(M));
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int i = 0; i < n_; ++i) acc += s->U(j, i) * (x[static_cast<size_t>(i)] * scale[static_cast<size_t>(i)]);
        tx[static_cast<size_t>(j)] = acc;
      }
      Mw.solve(tx.data(), mt.data());
      for (int i = 0; i < n_; ++i) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += s->U(j, i) * mt[static_cast<size_t>(j)];
        out[static_cast<size_t>(i)] = e1[static_cast<size_t>(i)] * x[static_cast<size_t>(i)] + scale[static_cast<size_t>(i)] * acc;
      }
      return out;
    }
    S.solve(x.data(), out.data());
    if (kind == 2 && M > 0) {
      std::vector<double> q(static_cast<size_t>(M)), mq(static_cast<size_t>(M));
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int i = 0; i < n_; ++i) acc += QUt(i, j) * out[static_cast<size_t>(i)];
        q[static_cast<size_t>(j)] = acc;
      }
      Mw.solve(q.data(), mq.data());
      for (int i = 0; i < n_; ++i) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += Z(i, j) * mq[static_cast<size_t>(j)];
        out[static_cast<size_t>(i)] += acc;
      }
    }
    return out;
  }
  double logdet_I_plus_WS() const {
    if (kind == 1) return logdet_fitc;
    double v = logdet_S + logdet_sigma;
    if (kind == 2 && s->basis.m() > 0) v += logdet_Mw - s->basis.llt.logdet();
    return v;
  }
  // latent cross covariance to a target and its prior variance (approximations.cpp:1121-1160,
  // 1202-1215, 1290-1355)
  std::pair<std::vector<double>, double> target_row(const Pt& q, int pred_m_v) const {
    const Model& m = *s;
    const orc_params& th = m.kernel.th;
    const int n_ = m.n, M = m.basis.m();
    if (kind == 1) {
      std::vector<double> up(static_cast<size_t>(M)), wp(static_cast<size_t>(M)), out(static_cast<size_t>(n_));
      for (int j = 0; j < M; ++j) up[static_cast<size_t>(j)] = m.kernel(m.basis.z[static_cast<size_t>(j)], q);
      m.basis.llt.solve(up.data(), wp.data());
      for (int i = 0; i < n_; ++i) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += m.U(j, i) * wp[static_cast<size_t>(j)];
        out[static_cast<size_t>(i)] = acc;
      }
      return {out, th.sigma1_2};
    }
    std::vector<double> resid(static_cast<size_t>(n_));
    std::vector<double> up(static_cast<size_t>(M)), wp(static_cast<size_t>(M)), wq(static_cast<size_t>(M));
    double u_smu = 0.0, rq = th.sigma1_2;
    if (kind == 2) {
      for (int i = 0; i < n_; ++i)
        resid[static_cast<size_t>(i)] = th.sigma1_2 - (M > 0 ? dot_seq(m.W.col(i), m.W.col(i), M) : 0.0);
      if (M > 0) {
        for (int j = 0; j < M; ++j) up[static_cast<size_t>(j)] = m.kernel(m.basis.z[static_cast<size_t>(j)], q);
        m.basis.llt.solve(up.data(), wp.data());
        m.basis.llt.lsolve(up.data(), wq.data());
        for (int j = 0; j < M; ++j) u_smu += up[static_cast<size_t>(j)] * wp[static_cast<size_t>(j)];
        rq -= dot_seq(wq.data(), wq.data(), M);
      }
    }
    const std::vector<int> N = kind == 0 ? target_nbrs(q, m, 1, 1.0, 1.0, nullptr, nullptr, 0.0, pred_m_v)
                                         : target_nbrs(q, m, 2, 1.0, 1.0, &resid, wq.data(), rq, pred_m_v);
    const int k = static_cast<int>(N.size());
    Mat C(k, k);
    std::vector<double> c(static_cast<size_t>(k)), A(static_cast<size_t>(k));
    for (int a = 0; a < k; ++a) {
      const int ja = N[static_cast<size_t>(a)];
      const Pt& pa = m.pts[static_cast<size_t>(ja)];
      double va = m.kernel(q, pa);
      if (kind == 2 && M > 0) va -= dot_seq(wq.data(), m.W.col(ja), M);
      c[static_cast<size_t>(a)] = va;
      for (int b = 0; b <= a; ++b) {
        const int jb = N[static_cast<size_t>(b)];
        double v = m.kernel(pa, m.pts[static_cast<size_t>(jb)]);
        if (kind == 2 && M > 0) v -= dot_seq(m.W.col(ja), m.W.col(jb), M);
        C(a, b) = v;
        C(b, a) = v;
      }
    }
    for (int a = 0; a < k; ++a) C(a, a) += 1e-10 * th.sigma1_2;
    Chol llt;
    if (!llt.compute(C))
      throw NumericError(kind == 0 ? "VecchiaLaplace: target conditioning block failed"
                                   : "VifLaplace: target conditioning block failed");
    if (k > 0) llt.solve(c.data(), A.data());
    double ac = 0.0;
    for (int a = 0; a < k; ++a) ac += A[static_cast<size_t>(a)] * c[static_cast<size_t>(a)];
    const double Dp = (kind == 0 ? th.sigma1_2 : rq) - ac;
    std::vector<double> sN(static_cast<size_t>(n_), 0.0);
    for (int a = 0; a < k; ++a) sN[static_cast<size_t>(N[static_cast<size_t>(a)])] = A[static_cast<size_t>(a)];
    std::vector<double> kvec = sigma_s_apply(m.nb, m.rows, sN.data());
    double var = (kind == 0 ? 0.0 : u_smu) + Dp;
    for (int a = 0; a < k; ++a) var += A[static_cast<size_t>(a)] * kvec[static_cast<size_t>(N[static_cast<size_t>(a)])];
    if (kind == 2 && M > 0)
      for (int i = 0; i < n_; ++i) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += m.U(j, i) * wp[static_cast<size_t>(j)];
        kvec[static_cast<size_t>(i)] += acc;
      }
    return {kvec, var};
  }
};

// latent_policy_nll (approximations.cpp:320-334)
double latent_policy_nll(Laplace& alg, double sigma2, const std::vector<double>& r) {
  if (!(sigma2 > 0.0)) throw NumericError("nll: the Gaussian path requires a positive nugget");
  const int n = static_cast<int>(r.size());
  const double w = 1.0 / sigma2;
  alg.prepare(std::vector<double>(static_cast<size_t>(n), w));
  const double logdet = n * std::log(sigma2) + alg.logdet_I_plus_WS();
  const std::vector<double> z = alg.solve(r);
  double rr = 0.0, rz = 0.0;
  for (int i = 0; i < n; ++i) {
    rr += r[static_cast<size_t>(i)] * r[static_cast<size_t>(i)];
    rz += r[static_cast<size_t>(i)] * z[static_cast<size_t>(i)];
  }
  const double quad = w * (rr - w * rz);
  return 0.5 * (logdet + quad + n * kLog2Pi);
}

// ZC-PTN observation model (laplace.cpp:25-91)
constexpr double kSqrt2 = 1.4142135623730951;
double norm_pdf(double z) { return std::exp(-0.5 * z * z - 0.5 * kLog2Pi); }
double norm_cdf(double z) { return 0.5 * std::erfc(-z / kSqrt2); }
double lower_tail_series(double z) {
  const double z2 = z * z, z4 = z2 * z2;
  return 1.0 - 1.0 / z2 + 3.0 / z4 - 15.0 / (z4 * z2) + 105.0 / (z4 * z4) - 945.0 / (z4 * z4 * z2);
}
double log_norm_cdf(double z) {
  if (z > -8.0) return std::log(norm_cdf(z));
  return -0.5 * z * z - 0.5 * kLog2Pi - std::log(-z) + std::log(lower_tail_series(z));
}
double inverse_mills(double z) {
  if (z > -8.0) return norm_pdf(z) / norm_cdf(z);
  return -z / lower_tail_series(z);
}
void validate_lik(double sigma, double lambda) {
  if (!(sigma > 0.0) || !std::isfinite(sigma)) throw ConfigError("LikelihoodParams: sigma must be > 0");
  if (!(lambda > 0.0) || !std::isfinite(lambda)) throw ConfigError("LikelihoodParams: lambda must be > 0");
}
double zcptn_loglik(double y, double mu, double sigma, double lambda) {
  if (y < 0.0) throw DataError("zcptn_loglik: negative precipitation amount");
  if (y == 0.0) return log_norm_cdf(-mu / sigma);
  const double g = std::pow(y, 1.0 / lambda);
  const double z = (g - mu) / sigma;
  return -0.5 * z * z - 0.5 * kLog2Pi - std::log(sigma) - std::log(lambda) - (1.0 - 1.0 / lambda) * std::log(y);
}
std::pair<double, double> zcptn_derivs(double y, double mu, double sigma, double lambda) {
  if (y < 0.0) throw DataError("zcptn_derivs: negative precipitation amount");
  if (y == 0.0) {
    const double z = -mu / sigma;
    const double h = inverse_mills(z);
    const double d1 = -h / sigma;
    const double d2 = (-z * h - h * h) / (sigma * sigma);
    return {d1, std::min(d2, 0.0)};
  }
  const double g = std::pow(y, 1.0 / lambda);
  return {(g - mu) / (sigma * sigma), -1.0 / (sigma * sigma)};
}

struct LapState {
  std::vector<double> mode, grad_at_mode, w;
  double log_marginal = 0.0;
  bool converged = false;
  int iterations = 0;
};

// laplace_marginal (laplace.cpp:115-203): Newton in (b, a = Sigma^{-1} b) with step halving
double laplace_marginal(Laplace& alg, const std::vector<double>& y, const std::vector<double>& offset, double sigma,
                        double lambda, const double* warm, LapState& st) {
  validate_lik(sigma, lambda);
  const int n = alg.n();
  auto value = [&](const std::vector<double>& b) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += zcptn_loglik(y[static_cast<size_t>(i)], offset[static_cast<size_t>(i)] + b[static_cast<size_t>(i)], sigma, lambda);
    return acc;
  };
  auto derivs = [&](const std::vector<double>& b, std::vector<double>& g, std::vector<double>& w) {
    g.resize(static_cast<size_t>(n));
    w.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      const auto d = zcptn_derivs(y[static_cast<size_t>(i)], offset[static_cast<size_t>(i)] + b[static_cast<size_t>(i)], sigma, lambda);
      g[static_cast<size_t>(i)] = d.first;
      w[static_cast<size_t>(i)] = std::max(-d.second, 0.0);
    }
  };
  auto dot = [&](const std::vector<double>& u, const std::vector<double>& v) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += u[static_cast<size_t>(i)] * v[static_cast<size_t>(i)];
    return acc;
  };
  std::vector<double> b(static_cast<size_t>(n), 0.0), a(static_cast<size_t>(n), 0.0), g, w;
  bool warm_nonzero = false;
  if (warm) {
    for (int i = 0; i < n; ++i) {
      b[static_cast<size_t>(i)] = warm[i];
      warm_nonzero = warm_nonzero || warm[i] != 0.0;
    }
  }
  if (warm_nonzero) {
    derivs(b, g, w);
    alg.prepare(w);
    std::vector<double> rhs(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) rhs[static_cast<size_t>(i)] = w[static_cast<size_t>(i)] * b[static_cast<size_t>(i)] + g[static_cast<size_t>(i)];
    const std::vector<double> bn = alg.solve(rhs);
    for (int i = 0; i < n; ++i) a[static_cast<size_t>(i)] = rhs[static_cast<size_t>(i)] - w[static_cast<size_t>(i)] * bn[static_cast<size_t>(i)];
    b = bn;
  }
  double psi = value(b) - 0.5 * dot(a, b);
  bool converged = false;
  int iter = 0;
  auto gap = [&]() {
    double mg = 0.0, md = 0.0;
    for (int i = 0; i < n; ++i) {
      mg = std::max(mg, std::abs(g[static_cast<size_t>(i)]));
      md = std::max(md, std::abs(g[static_cast<size_t>(i)] - a[static_cast<size_t>(i)]));
    }
    return md < 1e-6 * std::max(1.0, mg);
  };
  for (iter = 1; iter <= 100; ++iter) {
    derivs(b, g, w);
    if (gap()) {
      converged = true;
      break;
    }
    alg.prepare(w);
    std::vector<double> rhs(static_cast<size_t>(n)), an(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) rhs[static_cast<size_t>(i)] = w[static_cast<size_t>(i)] * b[static_cast<size_t>(i)] + g[static_cast<size_t>(i)];
    const std::vector<double> bn = alg.solve(rhs);
    for (int i = 0; i < n; ++i) an[static_cast<size_t>(i)] = rhs[static_cast<size_t>(i)] - w[static_cast<size_t>(i)] * bn[static_cast<size_t>(i)];
    double step = 1.0;
    bool accepted = false;
    for (int h = 0; h < 30; ++h) {
      std::vector<double> bt(static_cast<size_t>(n)), at(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) {
        bt[static_cast<size_t>(i)] = b[static_cast<size_t>(i)] + step * (bn[static_cast<size_t>(i)] - b[static_cast<size_t>(i)]);
        at[static_cast<size_t>(i)] = a[static_cast<size_t>(i)] + step * (an[static_cast<size_t>(i)] - a[static_cast<size_t>(i)]);
      }
      const double pt = value(bt) - 0.5 * dot(at, bt);
      if (pt >= psi - 1e-12 * std::abs(psi)) {
        b = bt;
        a = at;
        psi = pt;
        accepted = true;
        break;
      }
      step *= 0.5;
    }
    if (!accepted) break;
  }
  if (!converged) {
    derivs(b, g, w);
    converged = gap();
    if (!converged) throw NumericError("laplace_marginal: Newton did not converge in 100 iterations");
  }
  derivs(b, g, w);
  alg.prepare(w);
  const double lm = value(b) - 0.5 * dot(a, b) - 0.5 * alg.logdet_I_plus_WS();
  st.mode = b;
  st.grad_at_mode = a;
  st.w = w;
  st.log_marginal = lm;
  st.converged = converged;
  st.iterations = iter;
  return -lm;
}

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
double orc_exp(double x) { return std::exp(x); }
void orc_exp_array(long n, const double* x, double* out) {
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) out[i] = std::exp(x[i]);
}
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }
int orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
int orc_set_blas(const char* path, int threads) {
  return guarded([&] {
    if (!path || !*path) {
      g_blas = false;
      return;
    }
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) throw ConfigError(std::string("orc_set_blas: ") + dlerror());
    auto sym = [&](const char* a, const char* b) {
      void* f = dlsym(h, a);
      if (!f) f = dlsym(h, b);
      if (!f) throw ConfigError(std::string("orc_set_blas: missing ") + a);
      return f;
    };
    g_blas_fns.gemm = reinterpret_cast<dgemm_fn>(sym("scipy_dgemm_", "dgemm_"));
    g_blas_fns.syrk = reinterpret_cast<dsyrk_fn>(sym("scipy_dsyrk_", "dsyrk_"));
    g_blas_fns.trsm = reinterpret_cast<dtrsm_fn>(sym("scipy_dtrsm_", "dtrsm_"));
    g_blas_fns.set_threads = reinterpret_cast<void (*)(int)>(sym("scipy_openblas_set_num_threads", "openblas_set_num_threads"));
    if (threads > 0) g_blas_fns.set_threads(threads);
    g_blas = true;
  });
}

int orc_set_prune(int on) {
  g_prune = on != 0;
  return 0;
}

double orc_kernel_eval(const orc_params* p, double h, double u) {
  double v = std::numeric_limits<double>::quiet_NaN();
  guarded([&] { v = Kernel(*p).eval(h, u); });
  return v;
}
int orc_kernel_grad(const orc_params* p, double h, double u, double* g6) {
  return guarded([&] { Kernel(*p).grad(h, u, g6); });
}

// effective_ranges (covariance.cpp:231-254)
int orc_effective_ranges(const orc_params* p, double* tr, double* sr) {
  return guarded([&] {
    validate(*p);
    const double e = p->delta + p->beta;
    if (e <= 0.0 || p->a <= 0.0) {
      *tr = std::numeric_limits<double>::infinity();
    } else {
      const double T = std::pow(20.0, 1.0 / e);
      *tr = std::pow((T - 1.0) / p->a, 1.0 / (2.0 * p->alpha));
    }
    double lo = 0.0, hi = 1.0;
    while (matern(hi, p->nu) > 0.05) hi *= 2.0;
    while ((hi - lo) > 1e-10 * hi) {
      const double mid = 0.5 * (lo + hi);
      if (matern(mid, p->nu) > 0.05) lo = mid;
      else hi = mid;
    }
    *sr = 0.5 * (lo + hi) / p->c;
  });
}

// order_observations (dataset.cpp:81-114)
int orc_order_observations(int n, const double* t, uint64_t seed, int32_t* perm_out) {
  return guarded([&] {
    if (n <= 0) throw DataError("SpaceTimeDataset: empty dataset");
    std::vector<int> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return t[a] < t[b]; });
    std::mt19937_64 rng(mix_seed(seed, 0x0bde11));
    size_t bs = 0;
    for (size_t k = 1; k <= perm.size(); ++k) {
      const bool end = k == perm.size() || t[perm[k]] != t[perm[bs]];
      if (end) {
        for (size_t j = k - 1; j > bs; --j) {
          std::uniform_int_distribution<size_t> pick(bs, j);
          std::swap(perm[j], perm[pick(rng)]);
        }
        bs = k;
      }
    }
    for (int i = 0; i < n; ++i) perm_out[i] = perm[static_cast<size_t>(i)];
  });
}

double orc_dc_pair(const orc_params* p, double xa, double ya, double ta, double xb, double yb,
                   double tb) {
  double v = std::numeric_limits<double>::quiet_NaN();
  guarded([&] {
    Kernel k(*p);
    v = dc_metric(k, Pt{xa, ya, ta}, Pt{xb, yb, tb});
  });
  return v;
}

// correlation_neighbors (neighbors.cpp:318-322) == brute force on DcMetric.
// The selection kernel carries no lag table (estimation.cpp:200).
static void dc_search(int n, const double* x, const double* y, const double* t,
                      const orc_params* p, int m_v, int q0, int q1, int32_t* out, double* dist) {
  Kernel k(*p);
  const std::vector<Pt> pts = make_pts(n, x, y, t);
  const bool use_blocks = g_prune && time_sorted(pts);
  std::vector<std::pair<int, int>> blocks;
  if (use_blocks) blocks = time_blocks(pts);
#pragma omp parallel
  {
    std::vector<double> lb2(blocks.size());
#pragma omp for schedule(dynamic, 64)
    for (int i = q0; i < q1; ++i) {
      const Pt& pi = pts[static_cast<size_t>(i)];
      if (use_blocks)
        for (size_t b = 0; b < blocks.size(); ++b) {
          const double u = std::abs(pi.t - pts[static_cast<size_t>(blocks[b].first)].t);
          lb2[b] = 1.0 - k.live(u).pow_mE;  // |rho| <= T^{-(delta+beta)}
        }
      auto dist_fn = [&](int j) { return dc_metric(k, pi, pts[static_cast<size_t>(j)]); };
      topm_scan(i, m_v, dist_fn, use_blocks ? &blocks : nullptr, use_blocks ? &lb2 : nullptr,
                out + static_cast<size_t>(i - q0) * m_v, dist ? dist + static_cast<size_t>(i - q0) * m_v : nullptr);
    }
  }
}

int orc_dc_neighbors(int n, const double* x, const double* y, const double* t,
                     const orc_params* p, int m_v, int32_t* out, double* dist) {
  return guarded([&] { dc_search(n, x, y, t, p, m_v, 0, n, out, dist); });
}
int orc_dc_neighbors_range(int n, const double* x, const double* y, const double* t,
                           const orc_params* p, int m_v, int q0, int q1, int32_t* out) {
  return guarded([&] { dc_search(n, x, y, t, p, m_v, q0, q1, out, nullptr); });
}

// residual_neighbors (neighbors.cpp:51-83, 324-329) == brute force on DrMetric
int orc_dr_neighbors(int n, const double* x, const double* y, const double* t,
                     const orc_params* p, int M, const double* zx, const double* zy,
                     const double* zt, int m_v, int32_t* out, double* dist, double* W_out,
                     double* resid_out) {
  return guarded([&] {
    Kernel k(*p);
    const std::vector<Pt> pts = make_pts(n, x, y, t);
    std::vector<Pt> z;
    for (int j = 0; j < M; ++j) z.push_back({zx[j], zy[j], zt[j]});
    Basis basis(z, k);
    Mat W(M, n);
    if (M > 0) cross_and_whiten(basis, k, pts, nullptr, W, true);
    const double s1 = p->sigma1_2;
    const double tol = 1e-7 * s1;
    std::vector<double> resid(static_cast<size_t>(n));
    std::vector<char> degen(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      resid[static_cast<size_t>(i)] = M > 0 ? s1 - dot_seq(W.col(i), W.col(i), M) : s1;
      degen[static_cast<size_t>(i)] = resid[static_cast<size_t>(i)] <= tol;
    }
    if (W_out && M > 0) std::copy(W.a.begin(), W.a.end(), W_out);
    if (resid_out) std::copy(resid.begin(), resid.end(), resid_out);
#pragma omp parallel for schedule(dynamic, 16)
    for (int i = 0; i < n; ++i) {
      auto dist_fn = [&](int j) {
        if (degen[static_cast<size_t>(i)] || degen[static_cast<size_t>(j)]) return 1.0;
        double rho = k(pts[static_cast<size_t>(i)], pts[static_cast<size_t>(j)]);
        if (M > 0) rho -= dot_seq(W.col(i), W.col(j), M);
        const double rad = 1.0 - std::abs(rho) / std::sqrt(resid[static_cast<size_t>(i)] * resid[static_cast<size_t>(j)]);
        return std::sqrt(std::max(rad, 0.0));
      };
      topm_scan(i, m_v, dist_fn, nullptr, nullptr, out + static_cast<size_t>(i) * m_v,
                dist ? dist + static_cast<size_t>(i) * m_v : nullptr);
    }
  });
}

// residual_neighbors restricted to chosen query rows, with exact pruning so the large configurations
// (cfg3: 1e5 rows, cfg4: 1.1e6) are checkable.  The answer is the brute force's (orc_dr_neighbors); a
// candidate j is skipped only when a certified lower bound on its distance exceeds the query's current
// m-th distance by a margin, so (d, j) ties cannot be lost:
//   |rho_r(i,j)| = |k(i,j) - w_i.w_j| <= |k(i,j)| + sum_g |w_i[g]| |w_j[g]|       (Cauchy-Schwarz per group)
//   |k(i,j)|     <= s1 T(u)^{-(delta+beta)}                                         (Matern <= 1)
// The groups split the inducing points by time (and spatial cell): a query far from an inducing day has
// little weight in that day's group.  The computed dot differs from the exact one by at most
// gamma_M sum_a |w_i[a] w_j[a]|, covered by the (1 + 1e-9) factor; lb^2 carries a 1e-12 margin.
// Query lists are scanned backwards from i, time block by time block (blocks with a certified bound
// above the threshold are skipped whole), and candidates that survive every bound are evaluated exactly
// as in orc_dr_neighbors (kernel value minus the sequential-fma dot, sqrt(max(1 - |rho| / sqrt(r r), 0))).
static void dr_search_rows(int n, const double* x, const double* y, const double* t, const orc_params* p, int M,
                           const double* zx, const double* zy, const double* zt, int m_v, int nq, const int32_t* rows,
                           int32_t* out, double* dist, bool by_dist) {
  Kernel k(*p);
  const std::vector<Pt> pts = make_pts(n, x, y, t);
  if (!time_sorted(pts)) throw ConfigError("dr_search_rows: rows must be time ordered");
  bool integral = true;  // integer lags: the table equals the live factors bit for bit (covariance.cpp:115-123)
  double tmin = pts[0].t, tmax = pts[0].t;
  for (const Pt& q : pts) {
    integral = integral && q.t == std::nearbyint(q.t);
    tmin = std::min(tmin, q.t);
    tmax = std::max(tmax, q.t);
  }
  if (integral && tmax - tmin <= 200000.0) k.precompute(static_cast<int>(tmax - tmin) + 1);
  std::vector<Pt> z;
  for (int j = 0; j < M; ++j) z.push_back({zx[j], zy[j], zt[j]});
  // the candidates reach up to the last query row only
  int top = 0;
  for (int q = 0; q < nq; ++q) top = std::max(top, rows ? rows[q] + 1 : n);
  const std::vector<Pt> head(pts.begin(), pts.begin() + top);
  Basis basis(z, Kernel(*p));  // selection kernel: no lag table (estimation.cpp:200)
  Mat W(M, top);
  if (M > 0) cross_and_whiten(basis, Kernel(*p), head, nullptr, W, true);
  const double s1 = p->sigma1_2, tol = 1e-7 * s1;
  // inducing groups: distinct time (<= 8 quantile bins) x 3 x 3 spatial cells
  std::vector<int> grp(static_cast<size_t>(M), 0);
  int G = 1;
  if (M > 0) {
    std::vector<double> ts;
    for (const Pt& q : z) ts.push_back(q.t);
    std::sort(ts.begin(), ts.end());
    ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
    const int nt = std::min<int>(8, static_cast<int>(ts.size()));
    double x0 = zx[0], x1 = zx[0], y0 = zy[0], y1 = zy[0];
    for (int j = 0; j < M; ++j) {
      x0 = std::min(x0, zx[j]); x1 = std::max(x1, zx[j]);
      y0 = std::min(y0, zy[j]); y1 = std::max(y1, zy[j]);
    }
    for (int j = 0; j < M; ++j) {
      const long ti = std::lower_bound(ts.begin(), ts.end(), zt[j]) - ts.begin();
      const int tb = static_cast<int>(ti * nt / static_cast<long>(ts.size()));
      const int cx = x1 > x0 ? std::min(2, static_cast<int>(3.0 * (zx[j] - x0) / (x1 - x0))) : 0;
      const int cy = y1 > y0 ? std::min(2, static_cast<int>(3.0 * (zy[j] - y0) / (y1 - y0))) : 0;
      grp[static_cast<size_t>(j)] = (tb * 3 + cx) * 3 + cy;
    }
    G = nt * 9;
  }
  std::vector<double> resid(static_cast<size_t>(top)), gn(static_cast<size_t>(top) * G, 0.0), nrm(static_cast<size_t>(top));
  std::vector<char> degen(static_cast<size_t>(top));
#pragma omp parallel for schedule(static)
  for (int i = 0; i < top; ++i) {
    const double* w = W.col(i);
    resid[static_cast<size_t>(i)] = M > 0 ? s1 - dot_seq(w, w, M) : s1;
    degen[static_cast<size_t>(i)] = resid[static_cast<size_t>(i)] <= tol;
    double* g = &gn[static_cast<size_t>(i) * G];
    double tot = 0.0;
    for (int a = 0; a < M; ++a) g[grp[static_cast<size_t>(a)]] += w[a] * w[a];
    for (int q = 0; q < G; ++q) {
      tot += g[q];
      g[q] = std::sqrt(g[q]);
    }
    nrm[static_cast<size_t>(i)] = std::sqrt(tot);
  }
  // per time block: max |w_j| / sqrt(r_j) and min r_j over its non-degenerate rows
  const auto blocks = time_blocks(head);
  const size_t nb = blocks.size();
  std::vector<double> bA(nb, 0.0), bR(nb, std::numeric_limits<double>::infinity());
  for (size_t b = 0; b < nb; ++b)
    for (int j = blocks[b].first; j < blocks[b].second; ++j)
      if (!degen[static_cast<size_t>(j)]) {
        bA[b] = std::max(bA[b], nrm[static_cast<size_t>(j)] / std::sqrt(resid[static_cast<size_t>(j)]));
        bR[b] = std::min(bR[b], resid[static_cast<size_t>(j)]);
      }
  const double slack = 1.0 + 1e-9, margin = 1e-12;
#pragma omp parallel for schedule(dynamic, 4)
  for (int q = 0; q < nq; ++q) {
    const int i = rows ? rows[q] : q;
    int32_t* o = out + static_cast<size_t>(q) * m_v;
    double* od = dist ? dist + static_cast<size_t>(q) * m_v : nullptr;
    const int want = std::min(m_v, i);
    for (int a = 0; a < m_v; ++a) {
      o[a] = -1;
      if (od) od[a] = std::numeric_limits<double>::quiet_NaN();
    }
    if (want <= 0) continue;
    std::vector<std::pair<double, int>> heap;
    auto consider = [&](double d, int j) {
      const std::pair<double, int> c{d, j};
      if (static_cast<int>(heap.size()) < want) {
        heap.push_back(c);
        std::push_heap(heap.begin(), heap.end());
      } else if (c < heap.front()) {
        std::pop_heap(heap.begin(), heap.end());
        heap.back() = c;
        std::push_heap(heap.begin(), heap.end());
      }
    };
    const Pt& pi = pts[static_cast<size_t>(i)];
    const bool dq = degen[static_cast<size_t>(i)];
    const double ri = resid[static_cast<size_t>(i)], sri = std::sqrt(ri), ni = nrm[static_cast<size_t>(i)];
    const double* gi = &gn[static_cast<size_t>(i) * G];
    const double* wi = W.col(i);
    for (long b = static_cast<long>(nb) - 1; b >= 0; --b) {
      const int s = blocks[static_cast<size_t>(b)].first, e = std::min(blocks[static_cast<size_t>(b)].second, i);
      if (s >= e) continue;
      const double kb = s1 * k.factors(std::abs(pi.t - pts[static_cast<size_t>(s)].t)).pow_mE;
      const bool full = static_cast<int>(heap.size()) == want;
      if (full && !dq && bR[static_cast<size_t>(b)] < std::numeric_limits<double>::infinity()) {
        const double dm = heap.front().first;
        const double ub = (kb / (sri * std::sqrt(bR[static_cast<size_t>(b)])) + ni / sri * bA[static_cast<size_t>(b)]) * slack;
        // degenerate candidates sit at d = 1 and could only enter at dm == 1, where nothing is pruned
        if (1.0 - ub - margin > dm * dm) continue;
      }
      for (int j = e - 1; j >= s; --j) {
        if (dq || degen[static_cast<size_t>(j)]) {
          consider(1.0, j);
          continue;
        }
        const double rj = resid[static_cast<size_t>(j)], den = sri * std::sqrt(rj);
        if (static_cast<int>(heap.size()) == want) {
          const double dm2 = heap.front().first * heap.front().first;
          const double nj = nrm[static_cast<size_t>(j)];
          if (1.0 - (kb + ni * nj * slack) / den - margin > dm2) continue;
          const double kij = k(pi, pts[static_cast<size_t>(j)]);
          if (1.0 - (std::abs(kij) + ni * nj * slack) / den - margin > dm2) continue;
          const double* gj = &gn[static_cast<size_t>(j) * G];
          double gb = 0.0;
          for (int g = 0; g < G; ++g) gb += gi[g] * gj[g];
          if (1.0 - (std::abs(kij) + gb * slack) / den - margin > dm2) continue;
          const double rho = kij - (M > 0 ? dot_seq(wi, W.col(j), M) : 0.0);
          consider(std::sqrt(std::max(1.0 - std::abs(rho) / std::sqrt(ri * rj), 0.0)), j);
        } else {
          double rho = k(pi, pts[static_cast<size_t>(j)]);
          if (M > 0) rho -= dot_seq(wi, W.col(j), M);
          consider(std::sqrt(std::max(1.0 - std::abs(rho) / std::sqrt(ri * rj), 0.0)), j);
        }
      }
    }
    std::sort(heap.begin(), heap.end());
    if (od)
      for (size_t a = 0; a < heap.size(); ++a) od[a] = heap[a].first;
    std::vector<int> idx;
    for (const auto& h : heap) idx.push_back(h.second);
    if (!by_dist) std::sort(idx.begin(), idx.end());
    for (size_t a = 0; a < idx.size(); ++a) o[a] = idx[a];
  }
}

int orc_dr_neighbors_rows(int n, const double* x, const double* y, const double* t, const orc_params* p, int M,
                          const double* zx, const double* zy, const double* zt, int m_v, int nq, const int32_t* rows,
                          int32_t* out, double* dist, int by_dist) {
  return guarded([&] { dr_search_rows(n, x, y, t, p, M, zx, zy, zt, m_v, nq, rows, out, dist, by_dist != 0); });
}

// euclidean_neighbors (neighbors.cpp:257-316)
int orc_euclid_neighbors(int n, const double* x, const double* y, const double* t, int m_v,
                         double ss, double ts, int32_t* out) {
  return guarded([&] {
    if (!(ss > 0.0) || !(ts > 0.0)) throw ConfigError("euclidean_neighbors: scales must be positive");
    for (int i = 1; i < n; ++i)
      if (t[i] < t[i - 1]) throw ConfigError("euclidean_neighbors: dataset must be time-ordered");
    std::vector<double> sx(static_cast<size_t>(n)), sy(static_cast<size_t>(n)), st(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      sx[static_cast<size_t>(i)] = x[i] / ss;
      sy[static_cast<size_t>(i)] = y[i] / ss;
      st[static_cast<size_t>(i)] = t[i] / ts;
    }
    for (int k = 0; k < m_v; ++k) out[k] = -1;
#pragma omp parallel for schedule(dynamic, 64)
    for (int i = 1; i < n; ++i) {
      const int want = std::min(m_v, i);
      std::vector<std::pair<double, int>> heap;
      for (int j = i - 1; j >= 0; --j) {
        const double dt = st[static_cast<size_t>(i)] - st[static_cast<size_t>(j)];
        const double dt2 = dt * dt;
        if (static_cast<int>(heap.size()) == want && dt2 > heap.front().first) break;
        const double dx = sx[static_cast<size_t>(i)] - sx[static_cast<size_t>(j)];
        const double dy = sy[static_cast<size_t>(i)] - sy[static_cast<size_t>(j)];
        const double d2 = dt2 + dx * dx + dy * dy;
        const std::pair<double, int> c{d2, j};
        if (static_cast<int>(heap.size()) < want) {
          heap.push_back(c);
          std::push_heap(heap.begin(), heap.end());
        } else if (c < heap.front()) {
          std::pop_heap(heap.begin(), heap.end());
          heap.back() = c;
          std::push_heap(heap.begin(), heap.end());
        }
      }
      std::vector<int> idx;
      for (auto& h : heap) idx.push_back(h.second);
      std::sort(idx.begin(), idx.end());
      int32_t* o = out + static_cast<size_t>(i) * m_v;
      for (int k = 0; k < m_v; ++k) o[k] = k < static_cast<int>(idx.size()) ? idx[static_cast<size_t>(k)] : -1;
    }
  });
}

int orc_kmeanspp(const double* pts, int n, int d, int k, uint64_t seed, double* centers) {
  return guarded([&] {
    Mat P(n, d);
    std::copy(pts, pts + static_cast<size_t>(n) * d, P.a.begin());
    const Mat C = kmeanspp(P, k, seed);
    std::copy(C.a.begin(), C.a.end(), centers);
  });
}

// sts_kmeanspp (inducing.cpp:144-193)
int orc_sts_kmeanspp(int n, const double* x, const double* y, const double* t, int m,
                     uint64_t seed, int* m_s_out, int* m_t_out, double* out, int cap) {
  return guarded([&] {
    if (m < 1) throw ConfigError("sts_kmeanspp: m must be >= 1");
    std::set<double> ts;
    std::set<std::pair<double, double>> ss;
    for (int i = 0; i < n; ++i) {
      ts.insert(t[i]);
      ss.insert({x[i], y[i]});
    }
    Mat times(static_cast<int>(ts.size()), 1), locs(static_cast<int>(ss.size()), 2);
    int r = 0;
    for (double v : ts) times(r++, 0) = v;
    r = 0;
    for (const auto& s : ss) {
      locs(r, 0) = s.first;
      locs(r, 1) = s.second;
      ++r;
    }
    const double nt = static_cast<double>(times.r);
    int m_s = static_cast<int>(std::lround(std::sqrt(static_cast<double>(m) * n / (nt * nt))));
    int m_t = static_cast<int>(std::lround(std::sqrt(static_cast<double>(m) * nt * nt / n)));
    m_s = std::clamp(m_s, 1, std::min(locs.r, m));
    m_t = std::clamp(m_t, 1, std::min(times.r, m));
    const Mat sc = kmeanspp(locs, m_s, mix_seed(seed, 1));
    const Mat tc = kmeanspp(times, m_t, mix_seed(seed, 2));
    *m_s_out = m_s;
    *m_t_out = m_t;
    if (m_s * m_t > cap) throw ConfigError("sts_kmeanspp: output capacity too small");
    int o = 0;
    for (int js = 0; js < m_s; ++js)
      for (int jt = 0; jt < m_t; ++jt) {
        out[3 * o] = sc(js, 0);
        out[3 * o + 1] = sc(js, 1);
        out[3 * o + 2] = tc(jt, 0);
        ++o;
      }
  });
}

// joint_kmeanspp_inducing (inducing.cpp:117-142)
int orc_joint_kmeanspp(int n, const double* x, const double* y, const double* t, int m,
                       double ss, double ts, uint64_t seed, int* k_out, double* out, int cap) {
  return guarded([&] {
    if (!(ss > 0.0) || !(ts > 0.0)) throw ConfigError("joint_kmeanspp_inducing: scales must be positive");
    Mat S(n, 3);
    for (int i = 0; i < n; ++i) {
      S(i, 0) = x[i] / ss;
      S(i, 1) = y[i] / ss;
      S(i, 2) = t[i] / ts;
    }
    const int k = std::min(m, count_distinct_rows(S));
    const Mat C = kmeanspp(S, k, seed);
    if (k > cap) throw ConfigError("joint_kmeanspp: output capacity too small");
    *k_out = k;
    for (int j = 0; j < k; ++j) {
      out[3 * j] = C(j, 0) * ss;
      out[3 * j + 1] = C(j, 1) * ss;
      out[3 * j + 2] = C(j, 2) * ts;
    }
  });
}

int orc_inducing_logdet(int M, const double* zx, const double* zy, const double* zt,
                        const orc_params* p, int with_table_n, const double* data_t, double* logdet) {
  return guarded([&] {
    Kernel k(*p);
    if (with_table_n > 0) {
      std::vector<Pt> dp;
      for (int i = 0; i < with_table_n; ++i) dp.push_back({0, 0, data_t[i]});
      maybe_precompute_lags(k, dp);
    }
    std::vector<Pt> z;
    for (int j = 0; j < M; ++j) z.push_back({zx[j], zy[j], zt[j]});
    Basis b(z, k);
    *logdet = b.llt.logdet();
  });
}

int orc_build_rows(const orc_model* m, double* D_out, double* A_out) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    if (m->kind == 1) throw ConfigError("orc_build_rows: FITC has no Vecchia rows");
    std::copy(s.rows.D.begin(), s.rows.D.end(), D_out);
    if (A_out) std::copy(s.rows.A.begin(), s.rows.A.end(), A_out);
  });
}

int orc_fitc_diag(const orc_model* m, double* out) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    std::copy(s.fitc_diag.begin(), s.fitc_diag.end(), out);
  });
}

int orc_nll(const orc_model* m, const double* yv, int p, const double* X, const double* beta,
            double* out) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    const std::vector<double> r = residual(m->n, yv, p, X, beta);
    if (m->kind != 1 && m->policy != 1) {  // latent policy: nll through the Laplace algebra (approximations.cpp:348-349, 369-370)
      Laplace alg(s);
      *out = latent_policy_nll(alg, m->theta.sigma2, r);
      return;
    }
    *out = nll_model(s, r);
  });
}

int orc_nll_grad(const orc_model* m, const double* yv, int p, const double* X,
                 const double* beta, double* grad7) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    const std::vector<double> r = residual(m->n, yv, p, X, beta);
    if (m->kind == 0) grad_vecchia(s, r, grad7, nullptr);
    else if (m->kind == 1) grad_fitc(s, r, grad7, nullptr);
    else grad_vif(s, r, grad7, nullptr);
  });
}

// ZC-PTN helpers (laplace.cpp:25-91): out = {loglik, d1, d2}; tail = {norm_cdf, log_norm_cdf, inverse_mills}
int orc_zcptn(double y, double mu, double sigma, double lambda, double* out3) {
  return guarded([&] {
    validate_lik(sigma, lambda);
    out3[0] = zcptn_loglik(y, mu, sigma, lambda);
    const auto d = zcptn_derivs(y, mu, sigma, lambda);
    out3[1] = d.first;
    out3[2] = d.second;
  });
}
void orc_normal_tail(double z, double* out3) {
  out3[0] = norm_cdf(z);
  out3[1] = log_norm_cdf(z);
  out3[2] = inverse_mills(z);
}

// Laplace / ZC-PTN (laplace.cpp:115-259): the negative Laplace log-marginal, its state, and the
// latent predictive moments with the Monte Carlo draws on the observation scale
int orc_laplace_marginal(const orc_model* m, const double* yv, int p, const double* X, const double* beta,
                         double lik_sigma, double lik_lambda, const double* warm, double* nll_out, double* mode,
                         double* grad_at_mode, double* w_out, int* iterations) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    Laplace alg(s);
    const int n = m->n;
    std::vector<double> y(yv, yv + n), offset(static_cast<size_t>(n), 0.0);
    if (p > 0 && X && beta)
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < p; ++j) offset[static_cast<size_t>(i)] += X[static_cast<size_t>(i) + static_cast<size_t>(j) * n] * beta[j];
    LapState st;
    *nll_out = laplace_marginal(alg, y, offset, lik_sigma, lik_lambda, warm, st);
    for (int i = 0; i < n; ++i) {
      if (mode) mode[i] = st.mode[static_cast<size_t>(i)];
      if (grad_at_mode) grad_at_mode[i] = st.grad_at_mode[static_cast<size_t>(i)];
      if (w_out) w_out[i] = st.w[static_cast<size_t>(i)];
    }
    if (iterations) *iterations = st.iterations;
  });
}

int orc_zcptn_predict(const orc_model* m, const double* grad_at_mode, const double* w, int n_p, const double* qx,
                      const double* qy, const double* qt, const double* Xp, int p, const double* beta,
                      double lik_sigma, double lik_lambda, int pred_m_v, int n_samples, uint64_t seed,
                      double* mu_latent, double* var_latent, double* p_rain, double* amount_mean,
                      double* amount_median, double* samples, double* var_scale) {
  return guarded([&] {
    if (n_samples < 2) throw ConfigError("zcptn_predict: need at least two samples for scoring");
    Model s(m);
    build_model(s, m);
    Laplace alg(s);
    const int n = m->n;
    std::vector<double> wv(w, w + n), a(grad_at_mode, grad_at_mode + n);
    alg.prepare(wv);
    for (int pp = 0; pp < n_p; ++pp) {
      double off = 0.0;
      if (p > 0 && Xp && beta)
        for (int j = 0; j < p; ++j) off += Xp[static_cast<size_t>(pp) + static_cast<size_t>(j) * n_p] * beta[j];
      const Pt q{qx[pp], qy[pp], qt[pp]};
      const auto kr = alg.target_row(q, pred_m_v);
      const std::vector<double>& k = kr.first;
      double ka = 0.0, kwk = 0.0;
      std::vector<double> wk(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) {
        ka += k[static_cast<size_t>(i)] * a[static_cast<size_t>(i)];
        wk[static_cast<size_t>(i)] = wv[static_cast<size_t>(i)] * k[static_cast<size_t>(i)];
        kwk += k[static_cast<size_t>(i)] * wk[static_cast<size_t>(i)];
      }
      const std::vector<double> sw = alg.solve(wk);
      double wsw = 0.0;
      for (int i = 0; i < n; ++i) wsw += wk[static_cast<size_t>(i)] * sw[static_cast<size_t>(i)];
      const double mu_lat = off + ka;
      const double var_lat = std::max(kr.second - kwk + wsw, 0.0);
      mu_latent[pp] = mu_lat;
      var_latent[pp] = var_lat;
      if (var_scale) var_scale[pp] = std::abs(kr.second) + std::abs(kwk) + std::abs(wsw);
      const double s_tot = std::sqrt(lik_sigma * lik_sigma + var_lat);
      p_rain[pp] = 1.0 - norm_cdf(-mu_lat / s_tot);
      std::mt19937_64 rng(mix_seed(seed, static_cast<uint64_t>(pp)));
      std::normal_distribution<double> gauss(0.0, 1.0);
      const double sd = std::sqrt(var_lat);
      double acc = 0.0;
      std::vector<double> draws(static_cast<size_t>(n_samples));
      for (int t = 0; t < n_samples; ++t) {
        const double latent = mu_lat + sd * gauss(rng);
        const double zval = latent + lik_sigma * gauss(rng);
        const double amount = zval <= 0.0 ? 0.0 : std::pow(zval, lik_lambda);
        if (samples) samples[static_cast<size_t>(pp) + static_cast<size_t>(t) * n_p] = amount;
        draws[static_cast<size_t>(t)] = amount;
        acc += amount;
      }
      amount_mean[pp] = acc / n_samples;
      std::nth_element(draws.begin(), draws.begin() + n_samples / 2, draws.end());
      amount_median[pp] = draws[static_cast<size_t>(n_samples) / 2];
    }
  });
}

int orc_nll_grad_scale(const orc_model* m, const double* yv, int p, const double* X, const double* beta,
                       double* grad7, double* scale7) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    const std::vector<double> r = residual(m->n, yv, p, X, beta);
    if (m->kind == 0) grad_vecchia(s, r, grad7, scale7);
    else if (m->kind == 1) grad_fitc(s, r, grad7, scale7);
    else grad_vif(s, r, grad7, scale7);
  });
}

int orc_gls_beta(const orc_model* m, const double* yv, int p, const double* X, double* beta_out) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    if (m->kind != 1) require_obs(s, "gls_beta");
    const int n = m->n;
    if (p == 0) return;
    std::vector<std::vector<double>> SX(static_cast<size_t>(p));
    for (int j = 0; j < p; ++j) {
      std::vector<double> col(X + static_cast<size_t>(j) * n, X + static_cast<size_t>(j + 1) * n);
      SX[static_cast<size_t>(j)] = sigma_inv_apply(s, col);
    }
    std::vector<double> A(static_cast<size_t>(p) * p), b(static_cast<size_t>(p));
    for (int a = 0; a < p; ++a) {
      for (int c = 0; c < p; ++c) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += X[static_cast<size_t>(i) + static_cast<size_t>(a) * n] * SX[static_cast<size_t>(c)][static_cast<size_t>(i)];
        A[static_cast<size_t>(a) + static_cast<size_t>(c) * p] = acc;
      }
      double acc = 0.0;
      for (int i = 0; i < n; ++i) acc += SX[static_cast<size_t>(a)][static_cast<size_t>(i)] * yv[i];
      b[static_cast<size_t>(a)] = acc;
    }
    const std::vector<double> beta = spd_solve(p, A, b);
    std::copy(beta.begin(), beta.end(), beta_out);
  });
}

// predict (approximations.cpp:867-1080); metric_kind for Vecchia-family
// targets is taken from the neighbour sets' provenance passed in theta-less
// form: m->nbr provenance is not known here, so Vecchia uses d_c (1) and VIF
// uses d_r (2) -- the kinds the reference's correlation/residual searches set.
int orc_predict(const orc_model* m, const double* yv, int p, const double* X, const double* beta,
                int n_p, const double* qx, const double* qy, const double* qt, const double* Xp,
                int pred_m_v, double* mu, double* var) {
  return guarded([&] {
    Model s(m);
    build_model(s, m);
    const int n = m->n;
    const orc_params& th = m->theta;
    const std::vector<double> r = residual(n, yv, p, X, beta);
    std::vector<Pt> tg;
    for (int k = 0; k < n_p; ++k) tg.push_back({qx[k], qy[k], qt[k]});
    for (int k = 0; k < n_p; ++k) {
      double fe = 0.0;
      if (p > 0 && beta && Xp)
        for (int j = 0; j < p; ++j) fe += Xp[static_cast<size_t>(k) + static_cast<size_t>(j) * n_p] * beta[j];
      mu[k] = fe;
    }
    if (m->kind == 0) {
      require_obs(s, "predict");
      int code = 0;
      std::string err;
#pragma omp parallel for schedule(dynamic, 8)
      for (int pp = 0; pp < n_p; ++pp) {
        try {
          const Pt& q = tg[static_cast<size_t>(pp)];
          const std::vector<int> N = target_nbrs(q, s, 1, 1.0, 1.0, nullptr, nullptr, 0.0, pred_m_v);
          const int k = static_cast<int>(N.size());
          Mat C(k, k);
          std::vector<double> c(static_cast<size_t>(k)), rN(static_cast<size_t>(k)), A(static_cast<size_t>(k));
          for (int a = 0; a < k; ++a) {
            const Pt& pa = s.pts[static_cast<size_t>(N[static_cast<size_t>(a)])];
            c[static_cast<size_t>(a)] = s.kernel(q, pa);
            rN[static_cast<size_t>(a)] = r[static_cast<size_t>(N[static_cast<size_t>(a)])];
            for (int b = 0; b <= a; ++b) {
              double v = s.kernel(pa, s.pts[static_cast<size_t>(N[static_cast<size_t>(b)])]);
              if (a == b) v += th.sigma2;
              C(a, b) = v;
              C(b, a) = v;
            }
          }
          Chol llt;
          if (!llt.compute(C)) {
            for (int a = 0; a < k; ++a) C(a, a) += 1e-10 * th.sigma1_2;
            if (!llt.compute(C)) throw NumericError("predict: conditioning block not positive definite");
          }
          if (k > 0) llt.solve(c.data(), A.data());
          double ar = 0.0, ac = 0.0;
          for (int a = 0; a < k; ++a) {
            ar += A[static_cast<size_t>(a)] * rN[static_cast<size_t>(a)];
            ac += A[static_cast<size_t>(a)] * c[static_cast<size_t>(a)];
          }
          mu[pp] += ar;
          var[pp] = std::max(th.sigma1_2 + th.sigma2 - ac, 0.0);
        } catch (const NumericError& e) {
#pragma omp critical
          if (!code) {
            code = 4;
            err = e.what();
          }
        }
      }
      if (code) throw NumericError(err);
      return;
    }
    const int M = s.basis.m();
    const Mat& U = s.U;
    if (m->kind == 1) {
      std::vector<double> rl(static_cast<size_t>(n)), v(static_cast<size_t>(M)), Mv(static_cast<size_t>(M)), alpha(static_cast<size_t>(n));
      for (int i = 0; i < n; ++i) rl[static_cast<size_t>(i)] = r[static_cast<size_t>(i)] / s.lambda[static_cast<size_t>(i)];
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += U(j, i) * rl[static_cast<size_t>(i)];
        v[static_cast<size_t>(j)] = acc;
      }
      s.Mllt.solve(v.data(), Mv.data());
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += U(j, i) * Mv[static_cast<size_t>(j)];
        alpha[static_cast<size_t>(i)] = rl[static_cast<size_t>(i)] - (1.0 / s.lambda[static_cast<size_t>(i)]) * acc;
      }
      std::vector<double> Ua(static_cast<size_t>(M)), v2(static_cast<size_t>(M));
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += U(j, i) * alpha[static_cast<size_t>(i)];
        Ua[static_cast<size_t>(j)] = acc;
      }
      s.basis.llt.solve(Ua.data(), v2.data());
      Mat A1(M, M);
      if (g_blas) {
        blas_core(U, s.lambda, A1);
      } else {
#pragma omp parallel for schedule(static)
        for (int a = 0; a < M; ++a)
          for (int b = 0; b < M; ++b) {
            double acc = 0.0;
            for (int i = 0; i < n; ++i) acc += U(a, i) * (1.0 / s.lambda[static_cast<size_t>(i)]) * U(b, i);
            A1(a, b) = acc;
          }
      }
      const Mat MA1 = chol_solve_cols(s.Mllt, A1);
      Mat D12(M, M);
      if (g_blas) {
        D12 = A1;
        blas_gemm(false, false, -1.0, A1, MA1, 1.0, D12);
      } else {
#pragma omp parallel for schedule(static)
        for (int a = 0; a < M; ++a)
          for (int b = 0; b < M; ++b) {
            double acc = 0.0;
            for (int c = 0; c < M; ++c) acc += A1(a, c) * MA1(c, b);
            D12(a, b) = A1(a, b) - acc;
          }
      }
#pragma omp parallel for schedule(static)
      for (int pp = 0; pp < n_p; ++pp) {
        const Pt& q = tg[static_cast<size_t>(pp)];
        std::vector<double> up(static_cast<size_t>(M)), wp(static_cast<size_t>(M));
        for (int j = 0; j < M; ++j) up[static_cast<size_t>(j)] = s.kernel(s.basis.z[static_cast<size_t>(j)], q);
        double mu_l = 0.0;
        for (int j = 0; j < M; ++j) mu_l += up[static_cast<size_t>(j)] * v2[static_cast<size_t>(j)];
        mu[pp] += mu_l;
        s.basis.llt.solve(up.data(), wp.data());
        double shrink = 0.0;
        for (int a = 0; a < M; ++a) {
          double acc = 0.0;
          for (int b = 0; b < M; ++b) acc += D12(a, b) * wp[static_cast<size_t>(b)];
          shrink += wp[static_cast<size_t>(a)] * acc;
        }
        var[pp] = std::max(th.sigma1_2 + th.sigma2 - shrink, 0.0);
      }
      return;
    }
    // VIF
    require_obs(s, "predict");
    std::vector<double> resid(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) resid[static_cast<size_t>(i)] = th.sigma1_2 - (M > 0 ? dot_seq(s.W.col(i), s.W.col(i), M) : 0.0);
    const std::vector<double> ur = q_apply(s.nb, s.rows, r.data());
    std::vector<double> t(static_cast<size_t>(n), 0.0), yM(static_cast<size_t>(M));
    if (M > 0) {
      std::vector<double> w(static_cast<size_t>(M));
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += U(j, i) * ur[static_cast<size_t>(i)];
        w[static_cast<size_t>(j)] = acc;
      }
      s.Mllt.solve(w.data(), yM.data());
      for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int j = 0; j < M; ++j) acc += U(j, i) * yM[static_cast<size_t>(j)];
        t[static_cast<size_t>(i)] = acc;
      }
    }
    std::vector<double> z(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) z[static_cast<size_t>(i)] = r[static_cast<size_t>(i)] - t[static_cast<size_t>(i)];
    const std::vector<double> alpha = q_apply(s.nb, s.rows, z.data());
    std::vector<double> va(static_cast<size_t>(M));
    if (M > 0) {
      std::vector<double> Ua(static_cast<size_t>(M));
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += U(j, i) * alpha[static_cast<size_t>(i)];
        Ua[static_cast<size_t>(j)] = acc;
      }
      s.basis.llt.solve(Ua.data(), va.data());
    }
    int code = 0;
    std::string err;
#pragma omp parallel for schedule(dynamic, 8)
    for (int pp = 0; pp < n_p; ++pp) {
      try {
        const Pt& q = tg[static_cast<size_t>(pp)];
        std::vector<double> up(static_cast<size_t>(M)), wp(static_cast<size_t>(M)), wq(static_cast<size_t>(M));
        double u_smu = 0.0, rq = th.sigma1_2;
        if (M > 0) {
          for (int j = 0; j < M; ++j) up[static_cast<size_t>(j)] = s.kernel(s.basis.z[static_cast<size_t>(j)], q);
          s.basis.llt.solve(up.data(), wp.data());
          s.basis.llt.lsolve(up.data(), wq.data());
          for (int j = 0; j < M; ++j) u_smu += up[static_cast<size_t>(j)] * wp[static_cast<size_t>(j)];
          rq -= dot_seq(wq.data(), wq.data(), M);
        }
        const std::vector<int> N = target_nbrs(q, s, 2, 1.0, 1.0, &resid, wq.data(), rq, pred_m_v);
        const int k = static_cast<int>(N.size());
        Mat C(k, k);
        std::vector<double> c(static_cast<size_t>(k)), A(static_cast<size_t>(k));
        for (int a = 0; a < k; ++a) {
          const int ja = N[static_cast<size_t>(a)];
          const Pt& pa = s.pts[static_cast<size_t>(ja)];
          double va2 = s.kernel(q, pa);
          if (M > 0) va2 -= dot_seq(wq.data(), s.W.col(ja), M);
          c[static_cast<size_t>(a)] = va2;
          for (int b = 0; b <= a; ++b) {
            const int jb = N[static_cast<size_t>(b)];
            double v = s.kernel(pa, s.pts[static_cast<size_t>(jb)]);
            if (M > 0) v -= dot_seq(s.W.col(ja), s.W.col(jb), M);
            if (a == b) v += th.sigma2;
            C(a, b) = v;
            C(b, a) = v;
          }
        }
        Chol llt;
        if (!llt.compute(C)) {
          for (int a = 0; a < k; ++a) C(a, a) += 1e-10 * th.sigma1_2;
          if (!llt.compute(C)) throw NumericError("predict: residual conditioning block not positive definite");
        }
        if (k > 0) llt.solve(c.data(), A.data());
        double ac = 0.0;
        for (int a = 0; a < k; ++a) ac += A[static_cast<size_t>(a)] * c[static_cast<size_t>(a)];
        const double Dp = rq + th.sigma2 - ac;
        double mu_l = 0.0;
        if (M > 0)
          for (int j = 0; j < M; ++j) mu_l += up[static_cast<size_t>(j)] * va[static_cast<size_t>(j)];
        for (int a = 0; a < k; ++a) mu_l += A[static_cast<size_t>(a)] * z[static_cast<size_t>(N[static_cast<size_t>(a)])];
        mu[pp] += mu_l;
        std::vector<double> sN(static_cast<size_t>(n), 0.0);
        for (int a = 0; a < k; ++a) sN[static_cast<size_t>(N[static_cast<size_t>(a)])] = A[static_cast<size_t>(a)];
        const std::vector<double> cres = sigma_s_apply(s.nb, s.rows, sN.data());
        std::vector<double> cp(cres);
        std::vector<double> Utw(static_cast<size_t>(n), 0.0);
        if (M > 0) {
          for (int i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int j = 0; j < M; ++j) acc += U(j, i) * wp[static_cast<size_t>(j)];
            Utw[static_cast<size_t>(i)] = acc;
            cp[static_cast<size_t>(i)] += acc;
          }
        }
        double vprior = u_smu + Dp;
        for (int a = 0; a < k; ++a) vprior += A[static_cast<size_t>(a)] * cres[static_cast<size_t>(N[static_cast<size_t>(a)])];
        std::vector<double> qc(sN);
        if (M > 0) {
          const std::vector<double> qu = q_apply(s.nb, s.rows, Utw.data());
          for (int i = 0; i < n; ++i) qc[static_cast<size_t>(i)] += qu[static_cast<size_t>(i)];
        }
        double quad = 0.0;
        for (int i = 0; i < n; ++i) quad += cp[static_cast<size_t>(i)] * qc[static_cast<size_t>(i)];
        if (M > 0) {
          std::vector<double> mq(static_cast<size_t>(M)), Mmq(static_cast<size_t>(M));
          for (int j = 0; j < M; ++j) {
            double acc = 0.0;
            for (int i = 0; i < n; ++i) acc += U(j, i) * qc[static_cast<size_t>(i)];
            mq[static_cast<size_t>(j)] = acc;
          }
          s.Mllt.solve(mq.data(), Mmq.data());
          double qq = 0.0;
          for (int j = 0; j < M; ++j) qq += mq[static_cast<size_t>(j)] * Mmq[static_cast<size_t>(j)];
          quad -= qq;
        }
        var[pp] = std::max(vprior - quad, 0.0);
      } catch (const NumericError& e) {
#pragma omp critical
        if (!code) {
          code = 4;
          err = e.what();
        }
      }
    }
    if (code) throw NumericError(err);
  });
}

// DenseOracle (tests/oracles.cpp:10-112)
static long double matern_ld(long double x, long double nu) {
  if (x == 0.0L) return 1.0L;
  if (nu == 0.5L) return expl(-x);
  if (nu == 1.5L) return (1.0L + x) * expl(-x);
  if (nu == 2.5L) return (1.0L + x + x * x / 3.0L) * expl(-x);
  const double v = std::pow(2.0, 1.0 - static_cast<double>(nu)) / std::tgamma(static_cast<double>(nu)) *
                   std::pow(static_cast<double>(x), static_cast<double>(nu)) *
                   std::cyl_bessel_k(static_cast<double>(nu), static_cast<double>(x));
  return static_cast<long double>(std::isfinite(v) ? v : 0.0);
}
static long double gneiting_ld(long double h, long double u, const orc_params& th) {
  const long double a = th.a, alpha = th.alpha, beta = th.beta, delta = th.delta, c = th.c, s1 = th.sigma1_2;
  const long double T = a * powl(fabsl(u), 2.0L * alpha) + 1.0L;
  const long double E = delta + beta;
  const long double x = c * h / powl(T, beta / 2.0L);
  return s1 * powl(T, -E) * matern_ld(x, static_cast<long double>(th.nu));
}
static Mat dense_gram(const std::vector<Pt>& pts, const orc_params& th) {
  const int n = static_cast<int>(pts.size());
  Mat G(n, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j <= i; ++j) {
      const double v = static_cast<double>(gneiting_ld(static_cast<long double>(sdist(pts[static_cast<size_t>(i)], pts[static_cast<size_t>(j)])),
                                                       static_cast<long double>(tlag(pts[static_cast<size_t>(i)], pts[static_cast<size_t>(j)])), th));
      G(i, j) = v;
      G(j, i) = v;
    }
  for (int i = 0; i < n; ++i) G(i, i) += th.sigma2;
  return G;
}

int orc_dense_nll(int n, const double* x, const double* y, const double* t, const orc_params* p,
                  const double* yv, int pc, const double* X, const double* beta, double* out) {
  return guarded([&] {
    const std::vector<Pt> pts = make_pts(n, x, y, t);
    const Mat G = dense_gram(pts, *p);
    Chol c;
    if (!c.compute(G)) throw NumericError("dense oracle: Gram not positive definite");
    const std::vector<double> r = residual(n, yv, pc, X, beta);
    std::vector<double> s(static_cast<size_t>(n));
    c.solve(r.data(), s.data());
    double rs = 0.0;
    for (int i = 0; i < n; ++i) rs += r[static_cast<size_t>(i)] * s[static_cast<size_t>(i)];
    *out = 0.5 * (n * std::log(2.0 * M_PI) + c.logdet() + rs);
  });
}

int orc_dense_predict(int n, const double* x, const double* y, const double* t,
                      const orc_params* p, const double* yv, int n_p, const double* qx,
                      const double* qy, const double* qt, double* mu, double* var) {
  return guarded([&] {
    const std::vector<Pt> pts = make_pts(n, x, y, t);
    const Mat G = dense_gram(pts, *p);
    Chol c;
    if (!c.compute(G)) throw NumericError("dense oracle: Gram not positive definite");
    std::vector<double> s(static_cast<size_t>(n)), kv(static_cast<size_t>(n)), ks(static_cast<size_t>(n));
    c.solve(yv, s.data());
    for (int pp = 0; pp < n_p; ++pp) {
      const Pt q{qx[pp], qy[pp], qt[pp]};
      for (int i = 0; i < n; ++i)
        kv[static_cast<size_t>(i)] = static_cast<double>(gneiting_ld(static_cast<long double>(sdist(pts[static_cast<size_t>(i)], q)),
                                                                    static_cast<long double>(tlag(pts[static_cast<size_t>(i)], q)), *p));
      double m1 = 0.0;
      for (int i = 0; i < n; ++i) m1 += kv[static_cast<size_t>(i)] * s[static_cast<size_t>(i)];
      mu[pp] = m1;
      c.solve(kv.data(), ks.data());
      double kk = 0.0;
      for (int i = 0; i < n; ++i) kk += kv[static_cast<size_t>(i)] * ks[static_cast<size_t>(i)];
      var[pp] = p->sigma1_2 + p->sigma2 - kk;
    }
  });
}

// Test datasets of the reference suite, generated with the same libstdc++
// engines: kind 0 = random_ordered (test_neighbors.cpp:13-25, y uniform),
// kind 1 = make_random_dataset (test_approximations.cpp:16-32, y/X normal),
// kind 2 = grid_data (test_inducing.cpp:80-97, n = n_loc * n_times, unordered).
// Outputs are ordered by order_observations(seed) for kinds 0/1.
int orc_test_dataset(int kind, int n, uint64_t seed, int n_times, int p, double* x, double* y,
                     double* t, double* yv, double* X) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::normal_distribution<double> g(0.0, 1.0);
    std::vector<double> px, py, pt, pyv, pX;
    if (kind == 2) {
      const int n_loc = n;
      std::vector<double> xs, ys;
      for (int s2 = 0; s2 < n_loc; ++s2) {
        xs.push_back(u(rng));
        ys.push_back(u(rng));
      }
      int o = 0;
      for (int tt = 1; tt <= n_times; ++tt)
        for (int s2 = 0; s2 < n_loc; ++s2) {
          x[o] = xs[static_cast<size_t>(s2)];
          y[o] = ys[static_cast<size_t>(s2)];
          t[o] = static_cast<double>(tt);
          yv[o] = 0.0;
          ++o;
        }
      return;
    }
    pX.assign(static_cast<size_t>(n) * std::max(p, 0), 0.0);
    for (int i = 0; i < n; ++i) {
      const double a = u(rng), b = u(rng);
      const double tt = static_cast<double>(1 + static_cast<int>(u(rng) * n_times) % n_times);
      px.push_back(a);
      py.push_back(b);
      pt.push_back(tt);
      if (kind == 0) {
        pyv.push_back(u(rng));
      } else {
        pyv.push_back(g(rng));
        for (int j = 0; j < p; ++j) pX[static_cast<size_t>(i) + static_cast<size_t>(j) * n] = g(rng);
      }
    }
    std::vector<int32_t> perm(static_cast<size_t>(n));
    const int rc = orc_order_observations(n, pt.data(), seed, perm.data());
    if (rc) throw std::runtime_error(g_err);
    for (int i = 0; i < n; ++i) {
      const int s2 = perm[static_cast<size_t>(i)];
      x[i] = px[static_cast<size_t>(s2)];
      y[i] = py[static_cast<size_t>(s2)];
      t[i] = pt[static_cast<size_t>(s2)];
      yv[i] = pyv[static_cast<size_t>(s2)];
      for (int j = 0; j < p; ++j) X[static_cast<size_t>(i) + static_cast<size_t>(j) * n] = pX[static_cast<size_t>(s2) + static_cast<size_t>(j) * n];
    }
  });
}

}  // extern "C"

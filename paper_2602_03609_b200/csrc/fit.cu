// Maximum-likelihood fit driver on device-resident structures:
// the Gaussian path of stgp::fit (estimation.cpp:423-619) with its Transform
// (estimation.cpp:121-188), L-BFGS two-loop recursion (estimation.cpp:234-263), selection
// refresh on power-of-two iterations (neighbors.cpp:331-334, estimation.cpp:197-231),
// backtracking line search that halves the step on NumericError (estimation.cpp:564-586),
// GLS beta profiling (estimation.cpp:327-353, 520-525) and default_init (estimation.cpp:68-114).
//
// Host code sequences the engine's device phases; every objective value is a rebuild at theta
// plus the NLL, every gradient a rebuild plus the fused NLL + gradient (one build, where the
// reference builds twice).  The structure, its tiles and Ozaki workspace stay resident between
// iterations; a selection refresh replaces them.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <deque>
#include <limits>
#include <memory>
#include <numeric>
#include <random>
#include <vector>

#include "engine.hpp"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

double eval_value(stgp_structure* s, const Params& th, const double* y, const double* X, int p, const double* beta);
void eval_both(stgp_structure* s, const Params& th, const double* y, const double* X, int p, const double* beta,
               double* nll, double* grad);
void gls_beta_device(stgp_structure* s, const double* y_host, const double* X_host, int p, double* beta_out);
uint64_t mix_seed(uint64_t seed, uint64_t stream);

namespace {

constexpr double kBoundaryEps = 1e-6;
using vec = std::vector<double>;

double logit(double p) { return std::log(p / (1.0 - p)); }
double sigmoid(double z) {
  if (z >= 0.0) return 1.0 / (1.0 + std::exp(-z));
  const double e = std::exp(z);
  return e / (1.0 + e);
}
double dot(const vec& a, const vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double norm(const vec& a) { return std::sqrt(dot(a, a)); }

// Transform for the Gaussian likelihood (nugget present): z = (log s2, log s1, log a, log c,
// logit alpha, logit beta, log delta)   (estimation.cpp:126-147)
vec to_z(const Params& t) {
  return {std::log(std::max(t.sigma2, 1e-12)),
          std::log(t.sigma1_2),
          std::log(t.a),
          std::log(t.c),
          logit(std::clamp(t.alpha, kBoundaryEps, 1.0 - kBoundaryEps)),
          logit(std::clamp(t.beta, kBoundaryEps, 1.0 - kBoundaryEps)),
          std::log(std::max(t.delta, 1e-8))};
}
// CovarianceParams::validate (covariance.cpp:34-46): the reference's theta_of constructs a
// CovarianceParams, so a non-finite step raises ConfigError (not caught by the line search).
void validate_theta(const Params& t) {
  auto fail = [](const char* what) { config_error(std::string("CovarianceParams: ") + what); };
  if (!(t.sigma2 >= 0.0) || !std::isfinite(t.sigma2)) fail("sigma2 must be >= 0");
  if (!(t.sigma1_2 > 0.0) || !std::isfinite(t.sigma1_2)) fail("sigma1_2 must be > 0");
  if (!(t.a > 0.0) || !std::isfinite(t.a)) fail("a must be > 0");
  if (!(t.c > 0.0) || !std::isfinite(t.c)) fail("c must be > 0");
  if (!(t.alpha > 0.0 && t.alpha <= 1.0)) fail("alpha must be in (0, 1]");
  if (!(t.nu > 0.0) || !std::isfinite(t.nu)) fail("nu must be > 0");
  if (!(t.beta >= 0.0 && t.beta <= 1.0)) fail("beta must be in [0, 1]");
  if (!(t.delta >= 0.0) || !std::isfinite(t.delta)) fail("delta must be >= 0");
}
Params theta_of(const vec& z, double nu) {  // estimation.cpp:149-159
  Params t;
  t.sigma2 = std::exp(z[0]);
  t.sigma1_2 = std::exp(z[1]);
  t.a = std::exp(z[2]);
  t.c = std::exp(z[3]);
  t.alpha = std::clamp(sigmoid(z[4]), kBoundaryEps, 1.0);
  t.nu = nu;
  t.beta = std::clamp(sigmoid(z[5]), 0.0, 1.0);
  t.delta = std::exp(z[6]);
  validate_theta(t);
  return t;
}
vec dtheta_dz(const vec& z) {  // estimation.cpp:167-188
  const double sa = sigmoid(z[4]), sb = sigmoid(z[5]);
  return {std::exp(z[0]), std::exp(z[1]), std::exp(z[2]), std::exp(z[3]), sa * (1.0 - sa), sb * (1.0 - sb),
          std::exp(z[6])};
}

// L-BFGS, memory 10 (estimation.cpp:234-263)
struct Lbfgs {
  std::deque<std::pair<vec, vec>> pairs;
  void reset() { pairs.clear(); }
  void push(const vec& s, const vec& y) {
    if (dot(s, y) > 1e-12 * norm(s) * norm(y)) {
      pairs.emplace_back(s, y);
      if (pairs.size() > 10) pairs.pop_front();
    }
  }
  vec direction(const vec& g) const {
    vec q(g.size());
    for (size_t i = 0; i < g.size(); ++i) q[i] = -g[i];
    if (pairs.empty()) return q;
    vec alphas(pairs.size());
    for (size_t idx = pairs.size(); idx-- > 0;) {
      const auto& [s, y] = pairs[idx];
      const double rho = 1.0 / dot(s, y);
      alphas[idx] = rho * dot(s, q);
      for (size_t i = 0; i < q.size(); ++i) q[i] -= alphas[idx] * y[i];
    }
    const auto& [sl, yl] = pairs.back();
    const double gamma = dot(sl, yl) / dot(yl, yl);
    for (double& v : q) v *= gamma;
    for (size_t idx = 0; idx < pairs.size(); ++idx) {
      const auto& [s, y] = pairs[idx];
      const double rho = 1.0 / dot(s, y);
      const double bc = rho * dot(y, q);
      for (size_t i = 0; i < q.size(); ++i) q[i] += (alphas[idx] - bc) * s[i];
    }
    return q;
  }
};

struct Selection {  // estimation.cpp:191-195, owning the device objects
  stgp_neighbors* nb = nullptr;
  stgp_inducing* ind = nullptr;
  stgp_structure* s = nullptr;  // the approximation structure built on this selection
  Selection() = default;
  Selection(const Selection&) = delete;
  Selection& operator=(const Selection&) = delete;
  void release() {
    if (s) stgp_structure_destroy(s);
    if (nb) stgp_neighbors_destroy(nb);
    if (ind) stgp_inducing_destroy(ind);
    s = nullptr;
    nb = nullptr;
    ind = nullptr;
  }
  ~Selection() { release(); }
};

void check(int rc) {
  if (rc != STGP_OK) throw Error(rc, stgp_last_error());
}

stgp_params abi(const Params& p) {
  stgp_params o;
  std::memcpy(&o, &p, sizeof(o));
  return o;
}

// build_selection (estimation.cpp:197-231) plus the structure of the method on it
std::unique_ptr<Selection> build_selection(stgp_dataset* ds, const stgp_fit_config& cfg, const Params& th) {
  auto sel = std::make_unique<Selection>();
  const stgp_params t = abi(th);
  double tr = 0.0, sr = 0.0;
  check(stgp_effective_ranges(&t, &tr, &sr));
  const double ss = std::isfinite(sr) && sr > 0.0 ? sr : 1.0;
  const double ts = std::isfinite(tr) && tr > 0.0 ? tr : 1e6;
  switch (cfg.method) {
    case STGP_FIT_VECCHIA_EUCLID:
      check(stgp_euclidean_neighbors(ds, cfg.m_v, ss, ts, &sel->nb));
      check(stgp_build_vecchia(ds, &t, sel->nb, STGP_OBSERVATION, &sel->s));
      break;
    case STGP_FIT_VECCHIA_CORR:
      check(stgp_correlation_neighbors(ds, &t, cfg.m_v, &sel->nb));
      check(stgp_build_vecchia(ds, &t, sel->nb, STGP_OBSERVATION, &sel->s));
      break;
    case STGP_FIT_FITC_KMEANSPP:
      check(stgp_joint_kmeanspp_inducing(ds, cfg.m, ss, ts, cfg.seed, &sel->ind));
      check(stgp_build_fitc(ds, &t, sel->ind, &sel->s));
      break;
    case STGP_FIT_FITC_STS:
      check(stgp_sts_kmeanspp(ds, cfg.m, cfg.seed, &sel->ind));
      check(stgp_build_fitc(ds, &t, sel->ind, &sel->s));
      break;
    case STGP_FIT_VIF:
      check(stgp_sts_kmeanspp(ds, cfg.m, cfg.seed, &sel->ind));
      check(stgp_residual_neighbors(ds, &t, sel->ind, cfg.m_v, &sel->nb));
      check(stgp_build_vif(ds, &t, sel->ind, sel->nb, STGP_OBSERVATION, &sel->s));
      break;
    default:
      config_error("stgp_fit: unknown method");
  }
  return sel;
}

double quantile(std::vector<double>& v, double q) {  // estimation.cpp:59-66
  if (v.empty()) return 1.0;
  const auto k = static_cast<std::size_t>(std::min<double>(static_cast<double>(v.size()) - 1.0,
                                                           q * static_cast<double>(v.size())));
  std::nth_element(v.begin(), v.begin() + static_cast<long>(k), v.end());
  return v[k];
}

void validate_config(const stgp_fit_config& c) {  // estimation.cpp:18-35 (Gaussian likelihood)
  const bool vecchia = c.method == STGP_FIT_VECCHIA_EUCLID || c.method == STGP_FIT_VECCHIA_CORR ||
                       c.method == STGP_FIT_VIF;
  const bool inducing = c.method == STGP_FIT_FITC_KMEANSPP || c.method == STGP_FIT_FITC_STS ||
                        c.method == STGP_FIT_VIF;
  if (c.method < STGP_FIT_VECCHIA_EUCLID || c.method > STGP_FIT_VIF) config_error("unknown method");
  if (vecchia && c.m_v < 1) config_error("FitConfig: Vecchia-family methods need m_v >= 1");
  if (inducing && c.m < 1) config_error("FitConfig: inducing-point methods need m >= 1");
  if (c.max_iterations < 1) config_error("FitConfig: max_iterations >= 1");
  if (!(c.tol_objective > 0.0) || !(c.tol_gradient > 0.0)) config_error("FitConfig: tolerances must be positive");
  if (!(c.nu > 0.0)) config_error("FitConfig: nu must be positive");
  if (!(c.nu == 0.5 || c.nu == 1.5 || c.nu == 2.5))
    config_error("FitConfig: the Gaussian path needs analytic kernel gradients (nu in {0.5, 1.5, 2.5})");
}

// beta = (X^T X)^{-1} X^T y by a p x p Cholesky (the reference's LDLT of the same normal equations)
vec ols(const double* X, const double* y, int n, int p) {
  vec A(static_cast<size_t>(p) * p, 0.0), b(static_cast<size_t>(p), 0.0);
  for (int i = 0; i < p; ++i) {
    const double* xi = X + static_cast<size_t>(i) * n;
    for (int r = 0; r < n; ++r) b[i] += xi[r] * y[r];
    for (int j = 0; j <= i; ++j) {
      const double* xj = X + static_cast<size_t>(j) * n;
      double s = 0.0;
      for (int r = 0; r < n; ++r) s += xi[r] * xj[r];
      A[static_cast<size_t>(i) * p + j] = A[static_cast<size_t>(j) * p + i] = s;
    }
  }
  for (int j = 0; j < p; ++j) {  // in-place lower Cholesky
    double d = A[static_cast<size_t>(j) * p + j];
    for (int k = 0; k < j; ++k) d -= A[static_cast<size_t>(j) * p + k] * A[static_cast<size_t>(j) * p + k];
    if (!(d > 0.0)) numeric_error("fit: X^T X is singular");
    const double l = std::sqrt(d);
    A[static_cast<size_t>(j) * p + j] = l;
    for (int i = j + 1; i < p; ++i) {
      double s = A[static_cast<size_t>(i) * p + j];
      for (int k = 0; k < j; ++k) s -= A[static_cast<size_t>(i) * p + k] * A[static_cast<size_t>(j) * p + k];
      A[static_cast<size_t>(i) * p + j] = s / l;
    }
  }
  for (int i = 0; i < p; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= A[static_cast<size_t>(i) * p + k] * b[k];
    b[i] = s / A[static_cast<size_t>(i) * p + i];
  }
  for (int i = p - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = i + 1; k < p; ++k) s -= A[static_cast<size_t>(k) * p + i] * b[k];
    b[i] = s / A[static_cast<size_t>(i) * p + i];
  }
  return b;
}

Params default_init_host(const stgp_dataset* ds, const double* y, const double* X, int p, const stgp_fit_config& cfg) {
  const int n = ds->n;
  if (n < 10) data_error("default_init: need at least 10 observations");
  vec resid(y, y + n);
  if (p > 0) {
    const vec beta = ols(X, y, n, p);
    for (int r = 0; r < n; ++r)
      for (int j = 0; j < p; ++j) resid[r] -= X[static_cast<size_t>(j) * n + r] * beta[j];
  }
  double mean = 0.0;
  for (double v : resid) mean += v;
  mean /= n;
  double var = 0.0;
  for (double v : resid) var += (v - mean) * (v - mean);
  var /= std::max(1, n - 1);
  if (!(var > 0.0)) data_error("default_init: constant response");
  std::mt19937_64 rng(mix_seed(cfg.seed, 0x1417));
  const int sub = std::min(n, 1000);
  std::vector<int> rows(static_cast<size_t>(n));
  std::iota(rows.begin(), rows.end(), 0);
  std::shuffle(rows.begin(), rows.end(), rng);
  rows.resize(static_cast<size_t>(sub));
  std::vector<double> sd, td;
  for (int i = 0; i < sub; ++i)
    for (int j = 0; j < i; ++j) {
      const size_t a = static_cast<size_t>(rows[static_cast<size_t>(i)]), b = static_cast<size_t>(rows[static_cast<size_t>(j)]);
      const double dx = ds->hx[a] - ds->hx[b], dy = ds->hy[a] - ds->hy[b];
      const double s = std::sqrt(dx * dx + dy * dy), t = std::abs(ds->ht[a] - ds->ht[b]);
      if (s > 0.0) sd.push_back(s);
      if (t > 0.0) td.push_back(t);
    }
  const double alpha0 = 0.8;
  const double qs = quantile(sd, 0.10), qt = quantile(td, 0.10);
  Params th;
  th.sigma2 = 0.5 * var;
  th.sigma1_2 = 0.5 * var;
  th.a = std::clamp(1.0 / std::pow(std::max(qt, 1e-12), 2.0 * alpha0), 1e-8, 1e12);
  th.c = std::clamp(1.0 / std::max(qs, 1e-12), 1e-8, 1e12);
  th.alpha = alpha0;
  th.nu = cfg.nu;
  th.beta = 0.5;
  th.delta = 0.5;
  return th;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return STGP_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return STGP_ERR_INTERNAL;
  }
}

struct Trace {
  std::vector<stgp_trace_row> rows;
  void push(int it, double f, double gn, bool refresh) { rows.push_back({it, f, gn, refresh ? 1 : 0}); }
};

}  // namespace

}  // namespace stgp

extern "C" {

int stgp_default_init(const stgp_dataset* ds, const double* y, const double* X, int p, const stgp_fit_config* cfg,
                      stgp_params* out) {
  return stgp::guarded([&] {
    if (!ds || !y || !cfg || !out || (p > 0 && !X)) stgp::config_error("stgp_default_init: null argument");
    *out = stgp::abi(stgp::default_init_host(ds, y, X, p, *cfg));
  });
}

int stgp_fit(stgp_dataset* ds, const double* y, const double* X, int p, const stgp_fit_config* cfg_in,
             const stgp_params* init, stgp_params* theta_out, double* beta_out, double* final_nll, int* converged,
             stgp_trace_row* trace_out, int trace_cap, int* n_trace) {
  using namespace stgp;
  return guarded([&] {
    if (!ds || !y || !cfg_in || !theta_out || (p > 0 && !X)) config_error("stgp_fit: null argument");
    const stgp_fit_config cfg = *cfg_in;
    validate_config(cfg);
    Params theta0;
    if (init) std::memcpy(&theta0, init, sizeof(theta0));
    else theta0 = default_init_host(ds, y, X, p, cfg);
    theta0.nu = cfg.nu;  // nu is fixed per fit
    vec z = to_z(theta0);
    vec beta = p > 0 ? ols(X, y, ds->n, p) : vec();
    static const bool verbose = std::getenv("STGP_FIT_VERBOSE") != nullptr;  // per-evaluation log (stderr)
    auto log_eval = [&](const char* what, const vec& zz, double f) {
      if (!verbose) return;
      const Params t = theta_of(zz, cfg.nu);
      std::fprintf(stderr, "[fit] %s f=%.12g theta=(%g %g %g %g %g %g %g)\n", what, f, t.sigma2, t.sigma1_2, t.a, t.c,
                   t.alpha, t.beta, t.delta);
    };
    auto value = [&](stgp_structure* s, const vec& zz) {
      log_eval("value?", zz, std::nan(""));
      const double f = eval_value(s, theta_of(zz, cfg.nu), y, X, p, p > 0 ? beta.data() : nullptr);
      log_eval("value", zz, f);
      return f;
    };
    auto value_grad = [&](stgp_structure* s, const vec& zz, vec& g) {
      double f = 0.0;
      vec gt(7);
      log_eval("grad?", zz, std::nan(""));
      eval_both(s, theta_of(zz, cfg.nu), y, X, p, p > 0 ? beta.data() : nullptr, &f, gt.data());
      log_eval("grad", zz, f);
      const vec d = dtheta_dz(zz);
      g.assign(7, 0.0);
      for (int k = 0; k < 7; ++k) g[k] = gt[k] * d[k];
      return f;
    };
    std::unique_ptr<Selection> sel;
    Lbfgs lbfgs;
    double f = std::numeric_limits<double>::quiet_NaN();
    vec g;
    bool have_eval = false, done = false, conv = false;
    int terminal_refreshes = 0;
    Trace tr;
    auto refresh = [](int it) { return (it & (it - 1)) == 0; };  // neighbors.cpp:331-334
    for (int iter = 1; iter <= cfg.max_iterations && !done; ++iter) {
      bool refreshed = false;
      if (refresh(iter) || !have_eval) {
        if (verbose) std::fprintf(stderr, "[fit] iteration %d: selection refresh\n", iter);
        sel = build_selection(ds, cfg, theta_of(z, cfg.nu));
        refreshed = refresh(iter);
        vec gn;
        const double f_new = value_grad(sel->s, z, gn);
        if (have_eval && std::abs(f_new - f) > cfg.tol_objective * std::max(1.0, std::abs(f))) lbfgs.reset();
        f = f_new;
        g = gn;
        have_eval = true;
      }
      if (p > 0) {  // profile the GLS coefficients under the current covariance
        eval_value(sel->s, theta_of(z, cfg.nu), y, X, p, beta.data());  // build at theta
        gls_beta_device(sel->s, y, X, p, beta.data());
        f = value_grad(sel->s, z, g);
      }
      double gnorm = 0.0;
      for (double v : g) gnorm = std::max(gnorm, std::abs(v));
      tr.push(iter, f, gnorm, refreshed);
      const bool grad_ok = gnorm < cfg.tol_gradient;
      const bool obj_ok = tr.rows.size() >= 2 &&
                          std::abs(tr.rows[tr.rows.size() - 2].nll - f) < cfg.tol_objective * std::max(1.0, std::abs(f));
      if (grad_ok && obj_ok) {  // terminal refresh; resume only if it moved the likelihood
        auto rs = build_selection(ds, cfg, theta_of(z, cfg.nu));
        const double f_ref = value(rs->s, z);
        if (std::abs(f_ref - f) <= cfg.tol_objective * std::max(1.0, std::abs(f)) || terminal_refreshes >= 3) {
          sel = std::move(rs);
          f = f_ref;
          tr.push(iter, f, gnorm, true);
          conv = true;
          done = true;
          break;
        }
        sel = std::move(rs);
        f = value_grad(sel->s, z, g);
        lbfgs.reset();
        ++terminal_refreshes;
        tr.push(iter, f, gnorm, true);
        continue;
      }
      vec d = lbfgs.direction(g);
      if (dot(d, g) >= 0.0)
        for (size_t i = 0; i < d.size(); ++i) d[i] = -g[i];  // safeguard to a descent direction
      double step = 1.0;
      const double slope = dot(g, d);
      bool accepted = false;
      vec z_new(z.size());
      double f_new = f;
      for (int half = 0; half < 40; ++half) {
        for (size_t i = 0; i < z.size(); ++i) z_new[i] = z[i] + step * d[i];
        double f_try;
        try {
          f_try = value(sel->s, z_new);
        } catch (const Error& e) {
          if (e.code != kNumeric) throw;
          step *= 0.5;
          continue;
        }
        if (std::isfinite(f_try) && f_try <= f + 1e-4 * step * slope) {
          f_new = f_try;
          accepted = true;
          break;
        }
        step *= 0.5;
      }
      if (!accepted) {
        if (gnorm < cfg.tol_gradient * 10.0) conv = true;
        break;
      }
      vec g_new;
      value_grad(sel->s, z_new, g_new);
      vec sv(z.size()), yv(z.size());
      for (size_t i = 0; i < z.size(); ++i) {
        sv[i] = z_new[i] - z[i];
        yv[i] = g_new[i] - g[i];
      }
      lbfgs.push(sv, yv);
      z = z_new;
      f = f_new;
      g = g_new;
    }
    *theta_out = abi(theta_of(z, cfg.nu));
    if (beta_out && p > 0) std::copy(beta.begin(), beta.end(), beta_out);
    if (final_nll) *final_nll = f;
    if (converged) *converged = conv ? 1 : 0;
    if (n_trace) *n_trace = static_cast<int>(tr.rows.size());
    if (trace_out)
      for (int k = 0; k < std::min(trace_cap, static_cast<int>(tr.rows.size())); ++k) trace_out[k] = tr.rows[k];
    if (!std::isfinite(f)) numeric_error("fit: objective is not finite at the final iterate");
  });
}

}  // extern "C"

// C++ facade over the C ABI (stgp_b200.h) with the reference's names, argument
// meaning and exception types (proj/include/stgp/{types,covariance,neighbors,
// inducing,approximations}.hpp).  Header-only; link with libstgp_b200.so.
//
// Differences from the reference headers, all deliberate:
//  * no Eigen in the signatures: vectors are std::vector<double>, matrices are
//    column-major std::vector<double> with explicit row/column counts;
//  * structures are move-only handles to device-resident state; the fields the
//    reference tests read (B, D, fitc_diag) are downloaded on demand;
//  * the Laplace algebra (latent policy, ZC-PTN) factors Q + W densely on the device, so
//    Vecchia / VIF latent-policy structures are limited to n <= 40000 (the reference's
//    SimplicialLDLT is likewise a desk-scale method).
#ifndef STGP_B200_HPP
#define STGP_B200_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <algorithm>
#include <vector>

#include "stgp_b200.h"

namespace stgp_b200 {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == STGP_OK) return;
  const std::string msg = stgp_last_error();
  if (rc == STGP_ERR_CONFIG) throw ConfigError(msg);
  if (rc == STGP_ERR_DATA) throw DataError(msg);
  if (rc == STGP_ERR_NUMERIC) throw NumericError(msg);
  throw std::runtime_error(msg);
}

using CovarianceParams = stgp_params;  // field order of covariance.hpp:23-38
enum class DiagonalPolicy { kLatent = STGP_LATENT, kObservation = STGP_OBSERVATION };

template <class T, void (*Del)(T*)>
class Handle {
 public:
  Handle() = default;
  explicit Handle(T* p) : p_(p) {}
  Handle(Handle&& o) noexcept : p_(std::exchange(o.p_, nullptr)) {}
  Handle& operator=(Handle&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = std::exchange(o.p_, nullptr);
    }
    return *this;
  }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  ~Handle() { reset(); }
  T* get() const { return p_; }
  void reset() {
    if (p_) Del(p_);
    p_ = nullptr;
  }

 private:
  T* p_ = nullptr;
};

class Context {
 public:
  explicit Context(int device = 0) {
    stgp_ctx* c = nullptr;
    check(stgp_ctx_create(device, &c));
    h_ = Handle<stgp_ctx, stgp_ctx_destroy>(c);
  }
  stgp_ctx* get() const { return h_.get(); }
  void set_shard(int rank, int world) { check(stgp_ctx_set_shard(get(), rank, world)); }

 private:
  Handle<stgp_ctx, stgp_ctx_destroy> h_;
};

// SpaceTimeDataset (dataset.hpp:22-41), already in order_observations order
class SpaceTimeDataset {
 public:
  SpaceTimeDataset(Context& ctx, const std::vector<double>& x, const std::vector<double>& y,
                   const std::vector<double>& t)
      : n_(static_cast<int>(x.size())) {
    stgp_dataset* d = nullptr;
    check(stgp_dataset_create(ctx.get(), n_, x.data(), y.data(), t.data(), &d));
    h_ = Handle<stgp_dataset, stgp_dataset_destroy>(d);
  }
  void set_response(const std::vector<double>& resp, int p = 0, const std::vector<double>& X = {}) {
    check(stgp_dataset_set_response(get(), resp.data(), p, p > 0 ? X.data() : nullptr));
  }
  int n() const { return n_; }
  stgp_dataset* get() const { return h_.get(); }

 private:
  int n_;
  Handle<stgp_dataset, stgp_dataset_destroy> h_;
};

// order_observations permutation (dataset.cpp:81-114)
inline std::vector<int32_t> order_observations(const std::vector<double>& t, std::uint64_t seed) {
  std::vector<int32_t> perm(t.size());
  check(stgp_order_observations(static_cast<int>(t.size()), t.data(), seed, perm.data()));
  return perm;
}

// NeighborSets (neighbors.hpp:100-110)
class NeighborSets {
 public:
  explicit NeighborSets(stgp_neighbors* h) : h_(h) { check(stgp_neighbors_shape(h, &n_, &m_v_, &kind_)); }
  static NeighborSets from_sets(SpaceTimeDataset& ds, const std::vector<std::vector<int>>& sets, int m_v,
                                int kind = STGP_METRIC_DC) {
    std::vector<int32_t> flat(static_cast<size_t>(ds.n()) * m_v, -1);
    for (size_t i = 0; i < sets.size(); ++i)
      for (size_t a = 0; a < sets[i].size() && a < static_cast<size_t>(m_v); ++a) flat[i * m_v + a] = sets[i][a];
    stgp_neighbors* h = nullptr;
    check(stgp_neighbors_from_host(ds.get(), m_v, flat.data(), kind, &h));
    return NeighborSets(h);
  }
  std::vector<std::vector<int>> sets() const {
    std::vector<int32_t> flat(static_cast<size_t>(n_) * m_v_);
    check(stgp_neighbors_download(get(), flat.data(), nullptr));
    std::vector<std::vector<int>> out(static_cast<size_t>(n_));
    for (int i = 0; i < n_; ++i)
      for (int a = 0; a < m_v_; ++a)
        if (flat[static_cast<size_t>(i) * m_v_ + a] >= 0) out[static_cast<size_t>(i)].push_back(flat[static_cast<size_t>(i) * m_v_ + a]);
    return out;
  }
  int n() const { return n_; }
  int m_v() const { return m_v_; }
  stgp_neighbors* get() const { return h_.get(); }

 private:
  Handle<stgp_neighbors, stgp_neighbors_destroy> h_;
  int n_ = 0, m_v_ = 0, kind_ = 0;
};

// InducingSet (inducing.hpp:22-31)
class InducingSet {
 public:
  explicit InducingSet(stgp_inducing* h) : h_(h) { check(stgp_inducing_size(h, &M_, &m_s, &m_t)); }
  InducingSet(Context& ctx, const std::vector<double>& xyt_rowmajor) {
    stgp_inducing* h = nullptr;
    check(stgp_inducing_create(ctx.get(), static_cast<int>(xyt_rowmajor.size() / 3), xyt_rowmajor.data(), &h));
    h_ = Handle<stgp_inducing, stgp_inducing_destroy>(h);
    check(stgp_inducing_size(h, &M_, &m_s, &m_t));
  }
  std::vector<double> points() const {
    std::vector<double> out(static_cast<size_t>(M_) * 3);
    check(stgp_inducing_download(get(), out.data()));
    return out;
  }
  int size() const { return M_; }
  stgp_inducing* get() const { return h_.get(); }
  int m_s = 0, m_t = 0;

 private:
  Handle<stgp_inducing, stgp_inducing_destroy> h_;
  int M_ = 0;
};

inline NeighborSets euclidean_neighbors(SpaceTimeDataset& ds, int m_v, double space_scale, double time_scale) {
  stgp_neighbors* h = nullptr;
  check(stgp_euclidean_neighbors(ds.get(), m_v, space_scale, time_scale, &h));
  return NeighborSets(h);
}
inline NeighborSets correlation_neighbors(SpaceTimeDataset& ds, const CovarianceParams& theta, int m_v) {
  stgp_neighbors* h = nullptr;
  check(stgp_correlation_neighbors(ds.get(), &theta, m_v, &h));
  return NeighborSets(h);
}
inline NeighborSets residual_neighbors(SpaceTimeDataset& ds, const CovarianceParams& theta,
                                       const InducingSet& basis, int m_v) {
  stgp_neighbors* h = nullptr;
  check(stgp_residual_neighbors(ds.get(), &theta, basis.get(), m_v, &h));
  return NeighborSets(h);
}
inline InducingSet sts_kmeanspp(SpaceTimeDataset& ds, int m, std::uint64_t seed) {
  stgp_inducing* h = nullptr;
  check(stgp_sts_kmeanspp(ds.get(), m, seed, &h));
  return InducingSet(h);
}
inline InducingSet joint_kmeanspp_inducing(SpaceTimeDataset& ds, int m, double ss, double ts, std::uint64_t seed) {
  stgp_inducing* h = nullptr;
  check(stgp_joint_kmeanspp_inducing(ds.get(), m, ss, ts, seed, &h));
  return InducingSet(h);
}

// VecchiaStructure / FitcStructure / VifStructure (approximations.hpp:33-75)
class Structure {
 public:
  explicit Structure(stgp_structure* h, int n, int m_v) : h_(h), n_(n), m_v_(m_v) {}
  std::vector<double> D() const {
    std::vector<double> out(static_cast<size_t>(n_));
    check(stgp_structure_download_D(get(), out.data()));
    return out;
  }
  std::vector<double> A() const {  // B = I - A on N(i)
    std::vector<double> out(static_cast<size_t>(n_) * m_v_);
    check(stgp_structure_download_A(get(), out.data()));
    return out;
  }
  std::vector<double> fitc_diag() const {
    std::vector<double> out(static_cast<size_t>(n_));
    check(stgp_structure_download_fitc_diag(get(), out.data()));
    return out;
  }
  stgp_structure* get() const { return h_.get(); }
  int n() const { return n_; }

 private:
  Handle<stgp_structure, stgp_structure_destroy> h_;
  int n_, m_v_;
};

inline Structure build_vecchia(SpaceTimeDataset& ds, const CovarianceParams& theta, const NeighborSets& nb,
                               DiagonalPolicy policy = DiagonalPolicy::kLatent) {
  stgp_structure* h = nullptr;
  check(stgp_build_vecchia(ds.get(), &theta, nb.get(), static_cast<int>(policy), &h));
  return Structure(h, ds.n(), nb.m_v());
}
inline Structure build_fitc(SpaceTimeDataset& ds, const CovarianceParams& theta, const InducingSet& ind) {
  stgp_structure* h = nullptr;
  check(stgp_build_fitc(ds.get(), &theta, ind.get(), &h));
  return Structure(h, ds.n(), 1);
}
inline Structure build_vif(SpaceTimeDataset& ds, const CovarianceParams& theta, const InducingSet& ind,
                           const NeighborSets& nb, DiagonalPolicy policy = DiagonalPolicy::kLatent) {
  stgp_structure* h = nullptr;
  check(stgp_build_vif(ds.get(), &theta, ind.get(), nb.get(), static_cast<int>(policy), &h));
  return Structure(h, ds.n(), nb.m_v());
}

// y: length n; X: n x p column-major; beta: length p (may be empty)
inline double nll(Structure& s, const std::vector<double>& y, const std::vector<double>& X = {}, int p = 0,
                  const std::vector<double>& beta = {}) {
  double out = 0.0;
  check(stgp_nll(s.get(), y.data(), p ? X.data() : nullptr, p, p ? beta.data() : nullptr, &out));
  return out;
}
inline std::vector<double> nll_grad(Structure& s, const std::vector<double>& y, const std::vector<double>& X = {},
                                    int p = 0, const std::vector<double>& beta = {}) {
  std::vector<double> g(7);
  check(stgp_nll_grad(s.get(), y.data(), p ? X.data() : nullptr, p, p ? beta.data() : nullptr, g.data()));
  return g;
}
inline std::vector<double> gls_beta(Structure& s, const std::vector<double>& y, const std::vector<double>& X, int p) {
  std::vector<double> b(static_cast<size_t>(p));
  check(stgp_gls_beta(s.get(), y.data(), X.data(), p, b.data()));
  return b;
}

struct PredictiveDistribution {
  std::vector<double> mu, var;
};
inline PredictiveDistribution predict(Structure& s, const std::vector<double>& y, const std::vector<double>& X, int p,
                                      const std::vector<double>& beta, const std::vector<double>& targets_xyt,
                                      const std::vector<double>& X_p, int pred_m_v) {
  const int np = static_cast<int>(targets_xyt.size() / 3);
  PredictiveDistribution out{std::vector<double>(static_cast<size_t>(np)), std::vector<double>(static_cast<size_t>(np))};
  check(stgp_predict(s.get(), y.data(), p ? X.data() : nullptr, p, p ? beta.data() : nullptr, np, targets_xyt.data(),
                     p ? X_p.data() : nullptr, pred_m_v, out.mu.data(), out.var.data()));
  return out;
}

// LikelihoodParams / LaplaceState / ZcptnPrediction (covariance.hpp:41-48, laplace.hpp:37-62)
struct LikelihoodParams {
  double sigma = 1.0, lambda = 1.0;
};
struct LaplaceState {
  std::vector<double> mode, grad_at_mode, w;
  double log_marginal = 0.0;
  bool converged = false;
  int iterations = 0;
};
// laplace_marginal (laplace.hpp:47-53): {-log marginal, state}; latent-policy Vecchia / VIF or FITC
inline std::pair<double, LaplaceState> laplace_marginal(Structure& s, const std::vector<double>& y,
                                                        const std::vector<double>& X, int p,
                                                        const std::vector<double>& beta, const LikelihoodParams& lik,
                                                        const std::vector<double>* warm_start = nullptr) {
  const size_t n = y.size();
  LaplaceState st;
  st.mode.resize(n);
  st.grad_at_mode.resize(n);
  st.w.resize(n);
  double v = 0.0;
  check(stgp_laplace_marginal(s.get(), y.data(), p ? X.data() : nullptr, p, p ? beta.data() : nullptr, lik.sigma,
                              lik.lambda, warm_start && warm_start->size() == n ? warm_start->data() : nullptr, &v,
                              st.mode.data(), st.grad_at_mode.data(), st.w.data(), &st.iterations));
  st.log_marginal = -v;
  st.converged = true;  // a non-converged Newton raises NumericError (laplace.cpp:188-190)
  return {v, std::move(st)};
}
struct ZcptnPrediction {
  std::vector<double> mu_latent, var_latent, p_rain, amount_mean, amount_median;
  std::vector<double> samples;  // n_p x n_samples, column-major
};
// zcptn_predict (laplace.hpp:67-72)
inline ZcptnPrediction zcptn_predict(const LaplaceState& state, Structure& s, const std::vector<double>& targets_xyt,
                                     const std::vector<double>& X_p, int p, const std::vector<double>& beta,
                                     const LikelihoodParams& lik, int pred_m_v, int n_samples, std::uint64_t seed) {
  const int np = static_cast<int>(targets_xyt.size() / 3);
  ZcptnPrediction out;
  for (auto* v : {&out.mu_latent, &out.var_latent, &out.p_rain, &out.amount_mean, &out.amount_median})
    v->resize(static_cast<size_t>(np));
  out.samples.resize(static_cast<size_t>(np) * std::max(n_samples, 0));
  check(stgp_zcptn_predict(s.get(), state.grad_at_mode.data(), state.w.data(), np, targets_xyt.data(),
                           p ? X_p.data() : nullptr, p, p ? beta.data() : nullptr, lik.sigma, lik.lambda, pred_m_v,
                           n_samples, seed, out.mu_latent.data(), out.var_latent.data(), out.p_rain.data(),
                           out.amount_mean.data(), out.amount_median.data(), out.samples.data()));
  return out;
}

// FitConfig / TraceRow / FittedModel (estimation.hpp:23-83), Gaussian likelihood
using FitConfig = stgp_fit_config;
using TraceRow = stgp_trace_row;
struct FittedModel {
  CovarianceParams theta{};
  std::vector<double> beta;
  double final_nll = 0.0;
  bool converged = false;
  std::vector<TraceRow> trace;
};
inline FitConfig default_fit_config() {
  return FitConfig{STGP_FIT_VECCHIA_CORR, 30, 500, 200, 1e-8, 1e-5, 1.5, 0};
}
// default_init (estimation.cpp:68-114) on an ordered dataset
inline CovarianceParams default_init(const SpaceTimeDataset& ds, const std::vector<double>& y, const FitConfig& config,
                                     const std::vector<double>& X = {}, int p = 0) {
  CovarianceParams out{};
  check(stgp_default_init(ds.get(), y.data(), p ? X.data() : nullptr, p, &config, &out));
  return out;
}
// fit (estimation.cpp:423-619) on the ordered dataset (FittedModel.data); init nullptr -> default_init
inline FittedModel fit(SpaceTimeDataset& ds, const std::vector<double>& y, const FitConfig& config,
                       const CovarianceParams* init = nullptr, const std::vector<double>& X = {}, int p = 0) {
  FittedModel m;
  m.beta.assign(static_cast<size_t>(p), 0.0);
  std::vector<TraceRow> tr(4096);
  int conv = 0, ntr = 0;
  check(stgp_fit(ds.get(), y.data(), p ? X.data() : nullptr, p, &config, init, &m.theta, p ? m.beta.data() : nullptr,
                 &m.final_nll, &conv, tr.data(), static_cast<int>(tr.size()), &ntr));
  tr.resize(static_cast<size_t>(std::min(ntr, static_cast<int>(tr.size()))));
  m.trace = std::move(tr);
  m.converged = conv != 0;
  return m;
}

}  // namespace stgp_b200

#endif  // STGP_B200_HPP

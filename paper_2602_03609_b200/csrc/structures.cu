#include <cmath>
#include <algorithm>
#include <random>
// Structure builders and likelihood entry points (approximations.cpp:198-744).
// Vecchia lives here; the low-rank FITC/VIF algebra is in lowrank.cu.
#include <atomic>
#include <climits>
#include <cstring>

#include "comm.hpp"
#include "structure.hpp"
#include "lowrank_common.cuh"
#include "../../include/stgp_b200.h"

namespace stgp {

Params params_of(const stgp_params* th) {
  if (!th) config_error("null parameters");
  Params p;
  std::memcpy(&p, th, sizeof(p));
  validate_params(p);
  return p;
}

stgp_structure* new_structure(stgp_dataset* ds, int kind, const Params& th, const stgp_neighbors* nb, int policy) {
  if (!ds) config_error("null dataset");
  auto s = std::make_unique<stgp_structure>();
  s->ds = ds;
  s->kind = kind;
  s->policy = policy;
  s->th = th;
  s->n = ds->n;
  shard_rows(ds->ctx, s->n, s->row_begin, s->row_end);
  cudaStream_t st = ds->ctx->stream;
  if (nb) {
    if (nb->n != ds->n) config_error("build: neighbor sets inconsistent with the dataset");
    s->m_v = nb->m_v;
    s->nbr_kind = nb->kind;
    s->nbr_ss = nb->ss;
    s->nbr_ts = nb->ts;
    s->nbr.alloc(static_cast<size_t>(s->n) * s->m_v);
    STGP_CUDA(cudaMemcpyAsync(s->nbr.get(), nb->idx.get(), static_cast<size_t>(s->n) * s->m_v * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, st));
  } else {
    s->m_v = 1;
    std::vector<int32_t> none(static_cast<size_t>(s->n), -1);
    s->nbr.upload(none.data(), none.size(), st);
  }
  s->A.alloc(static_cast<size_t>(s->n) * s->m_v);
  s->D.alloc(static_cast<size_t>(s->n));
  s->A.zero(st);
  s->D.zero(st);
  s->ti.T = ds->Tdata;
  s->ti.build();
  s->ti_dirty = true;
  s->fail.alloc(1);
  return s.release();
}

static void require_obs(const stgp_structure* s, const char* what) {
  if (s->policy != STGP_OBSERVATION)
    numeric_error(std::string(what) +
                  ": analytic gradient is defined for the observation-policy structure driven by the optimizer");
}

// ---- Vecchia ----
void vecchia_build(stgp_structure* s) {
  prepare_tables(s);
  const double nug = s->policy == STGP_OBSERVATION ? s->th.sigma2 : 0.0;
  run_rows(s, kModeBuild, nullptr, 0, nug);
  s->built = true;
}

double vecchia_nll(stgp_structure* s) {
  if (s->policy != STGP_OBSERVATION) {  // approximations.cpp:348-349: through the Laplace algebra
    laplace_release(s);
    const double v = latent_policy_nll_dev(s);
    laplace_release(s);
    return v;
  }
  stgp_ctx* ctx = s->ds->ctx;
  const int rows = s->row_end - s->row_begin;
  const int blocks = std::max(1, std::min(ceil_div(rows, 256), ctx->num_sms * 4));
  s->red.ensure(blocks, 1);
  launch_nll_stored(s, blocks, nullptr);
  std::vector<double> tot = s->red.finish(ctx, blocks, 1);
  allreduce_host(ctx, tot);
  return 0.5 * (tot[0] + nll_const(s->n));
}

void vecchia_nll_grad(stgp_structure* s, double* nll, double* grad) {
  require_obs(s, "nll_grad");
  require_analytic_grad(s->th);
  prepare_tables(s);
  std::vector<double> tot = run_rows(s, kModeGrad, nullptr, 0, s->th.sigma2);
  allreduce_host(s->ds->ctx, tot);
  if (nll) *nll = 0.5 * (tot[0] + nll_const(s->n));
  if (grad)
    for (int q = 0; q < 7; ++q) grad[q] = tot[1 + q];
  s->built = true;
}

}  // namespace stgp

using namespace stgp;

stgp_structure::~stgp_structure() { stgp::laplace_release(this); }

stgp_structure::stgp_structure() {
  static std::atomic<uint64_t> next{1};
  uid = next.fetch_add(1);
}

namespace {
template <class F>
int guarded(F&& f) {
  try {
    f();
    return STGP_OK;
  } catch (const stgp::Error& e) {
    stgp::g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    stgp::g_last_error = e.what();
    return STGP_ERR_INTERNAL;
  }
}
}  // namespace

// declared in lowrank.cu
namespace stgp {
void lowrank_setup(stgp_structure* s, const stgp_inducing* ind);
void fitc_build(stgp_structure* s);
void vif_build(stgp_structure* s);
double lowrank_nll(stgp_structure* s);
void lowrank_nll_grad(stgp_structure* s, double* nll, double* grad);
void lowrank_predict(stgp_structure* s, int n_p, const double* txyt, int pred_m_v, double* mu, double* var);
void vecchia_predict(stgp_structure* s, int n_p, const double* txyt, int pred_m_v, double* mu, double* var);
void gls_beta_device(stgp_structure* s, const double* y_host, const double* X_host, int p, double* beta_out);
}  // namespace stgp

namespace stgp {
double lowrank_nll(stgp_structure* s);
// Objective value at theta: rebuild + NLL (the fit driver's line search, estimation.cpp:358-379)
double eval_value(stgp_structure* s, const Params& th, const double* y, const double* X, int p, const double* beta) {
  validate_params(th);
  s->th = th;
  compute_residual(s, y, X, p, beta);
  if (s->kind == STGP_VECCHIA) {
    vecchia_build(s);
    return vecchia_nll(s);
  }
  if (s->kind == STGP_FITC) fitc_build(s);
  else vif_build(s);
  return lowrank_nll(s);
}
// Value and gradient at theta: one rebuild + the fused NLL and gradient
void eval_both(stgp_structure* s, const Params& th, const double* y, const double* X, int p, const double* beta,
               double* nll, double* grad) {
  validate_params(th);
  s->th = th;
  compute_residual(s, y, X, p, beta);
  if (s->kind == STGP_VECCHIA) {
    vecchia_nll_grad(s, nll, grad);
  } else {
    if (s->kind == STGP_FITC) fitc_build(s);
    else vif_build(s);
    lowrank_nll_grad(s, nll, grad);
  }
}
}  // namespace stgp

extern "C" {

int stgp_build_vecchia(stgp_dataset* ds, const stgp_params* theta, const stgp_neighbors* nb, int policy,
                       stgp_structure** out) {
  return guarded([&] {
    if (!out || !nb) config_error("stgp_build_vecchia: null argument");
    std::unique_ptr<stgp_structure> s(new_structure(ds, STGP_VECCHIA, params_of(theta), nb, policy));
    vecchia_build(s.get());
    *out = s.release();
  });
}

int stgp_build_fitc(stgp_dataset* ds, const stgp_params* theta, const stgp_inducing* ind, stgp_structure** out) {
  return guarded([&] {
    if (!out || !ind) config_error("stgp_build_fitc: null argument");
    if (ind->M() < 1) config_error("build_fitc: need at least one inducing point");
    std::unique_ptr<stgp_structure> s(new_structure(ds, STGP_FITC, params_of(theta), nullptr, STGP_OBSERVATION));
    lowrank_setup(s.get(), ind);
    fitc_build(s.get());
    *out = s.release();
  });
}

int stgp_build_vif(stgp_dataset* ds, const stgp_params* theta, const stgp_inducing* ind, const stgp_neighbors* nb,
                   int policy, stgp_structure** out) {
  return guarded([&] {
    if (!out || !ind || !nb) config_error("stgp_build_vif: null argument");
    std::unique_ptr<stgp_structure> s(new_structure(ds, STGP_VIF, params_of(theta), nb, policy));
    lowrank_setup(s.get(), ind);
    vif_build(s.get());
    *out = s.release();
  });
}

void stgp_structure_destroy(stgp_structure* s) { delete s; }

int stgp_structure_download_D(const stgp_structure* s, double* D) {
  return guarded([&] {
    if (s->kind == STGP_FITC) config_error("FITC structures have no Vecchia factor D");
    s->D.download(D, static_cast<size_t>(s->n), s->ds->ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(s->ds->ctx->stream));
  });
}

int stgp_structure_download_A(const stgp_structure* s, double* A) {
  return guarded([&] {
    if (s->kind == STGP_FITC) config_error("FITC structures have no Vecchia factor B");
    s->A.download(A, static_cast<size_t>(s->n) * s->m_v, s->ds->ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(s->ds->ctx->stream));
  });
}

int stgp_structure_download_fitc_diag(const stgp_structure* s, double* out) {
  return guarded([&] {
    if (s->kind != STGP_FITC) config_error("only FITC structures carry fitc_diag");
    s->lr.fitc_diag.download(out, static_cast<size_t>(s->n), s->ds->ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(s->ds->ctx->stream));
  });
}

int stgp_nll(stgp_structure* s, const double* y, const double* X, int p, const double* beta, double* out) {
  return guarded([&] {
    if (!s || !out) config_error("stgp_nll: null argument");
    compute_residual(s, y, X, p, beta);
    if (s->kind == STGP_VECCHIA) *out = vecchia_nll(s);
    else *out = lowrank_nll(s);
  });
}

int stgp_nll_grad(stgp_structure* s, const double* y, const double* X, int p, const double* beta, double* grad) {
  return guarded([&] {
    if (!s || !grad) config_error("stgp_nll_grad: null argument");
    compute_residual(s, y, X, p, beta);
    if (s->kind == STGP_VECCHIA) vecchia_nll_grad(s, nullptr, grad);
    else lowrank_nll_grad(s, nullptr, grad);
  });
}

int stgp_nll_and_grad(stgp_structure* s, const double* y, const double* X, int p, const double* beta, double* nll,
                      double* grad) {
  return guarded([&] {
    if (!s) config_error("stgp_nll_and_grad: null argument");
    compute_residual(s, y, X, p, beta);
    if (s->kind == STGP_VECCHIA) vecchia_nll_grad(s, nll, grad);
    else lowrank_nll_grad(s, nll, grad);
  });
}

int stgp_eval(stgp_structure* s, const stgp_params* theta, const double* y, const double* X, int p,
              const double* beta, double* nll, double* grad) {
  return guarded([&] {
    if (!s) config_error("stgp_eval: null structure");
    s->th = params_of(theta);
    compute_residual(s, y, X, p, beta);
    if (s->kind == STGP_VECCHIA) {
      vecchia_nll_grad(s, nll, grad);
    } else {
      if (s->kind == STGP_FITC) fitc_build(s);
      else vif_build(s);
      lowrank_nll_grad(s, nll, grad);
    }
  });
}

int stgp_gls_beta(stgp_structure* s, const double* y, const double* X, int p, double* beta_out) {
  return guarded([&] {
    if (!s || !beta_out) config_error("stgp_gls_beta: null argument");
    if (s->kind != STGP_FITC && s->policy != STGP_OBSERVATION)
      numeric_error("gls_beta: requires the observation-policy structure");
    if (p <= 0) return;
    if (s->ds->ctx->world > 1) config_error("gls_beta: run on an unsharded context (stgp_ctx_set_shard(ctx, 0, 1))");
    gls_beta_device(s, y, X, p, beta_out);
  });
}

int stgp_predict(stgp_structure* s, const double* y, const double* X, int p, const double* beta, int n_p,
                 const double* txyt, const double* Xp, int pred_m_v, double* mu, double* var) {
  return guarded([&] {
    if (!s || !mu || !var) config_error("stgp_predict: null argument");
    if (s->kind != STGP_FITC && s->policy != STGP_OBSERVATION)
      numeric_error("predict: requires the observation-policy structure");
    compute_residual(s, y, X, p, beta);
    if (n_p <= 0) return;
    if (s->kind != STGP_VECCHIA && s->ds->ctx->world > 1)
      config_error("predict: FITC/VIF prediction runs on an unsharded context (stgp_ctx_set_shard(ctx, 0, 1))");
    if (s->kind == STGP_VECCHIA) vecchia_predict(s, n_p, txyt, pred_m_v, mu, var);
    else lowrank_predict(s, n_p, txyt, pred_m_v, mu, var);
    // fixed effect X_p beta (approximations.cpp:806-812)
    if (p > 0 && beta && Xp)
      for (int k = 0; k < n_p; ++k) {
        double fe = 0.0;
        for (int j = 0; j < p; ++j) fe += Xp[static_cast<size_t>(k) + static_cast<size_t>(j) * n_p] * beta[j];
        mu[k] += fe;
      }
  });
}

// laplace_marginal (laplace.cpp:115-203) with the ZC-PTN likelihood on a latent-policy structure (FITC: any)
int stgp_laplace_marginal(stgp_structure* s, const double* y, const double* X, int p, const double* beta,
                          double lik_sigma, double lik_lambda, const double* warm, double* nll_out, double* mode,
                          double* grad_at_mode, double* w, int* iterations) {
  return guarded([&] {
    if (!s || !y || !nll_out) config_error("stgp_laplace_marginal: null argument");
    compute_residual(s, y, X, p, beta);  // ywork = y, r = y - X beta
    DevBuf<double> off(static_cast<size_t>(s->n));
    vsub(s->ds->ctx, s->n, s->ywork.get(), s->r.get(), off.get());  // X beta
    laplace_release(s);
    *nll_out = laplace_marginal_dev(s, y, off.get(), lik_sigma, lik_lambda, warm, mode, grad_at_mode, w, iterations);
    laplace_release(s);
  });
}

// zcptn_predict (laplace.cpp:205-259): latent moments on the device from the Laplace state, then the
// occurrence probability and the Monte Carlo amounts with the reference's per-target RNG streams
// (mt19937_64(mix_seed(seed, p)), std::normal_distribution) on the host
int stgp_zcptn_predict(stgp_structure* s, const double* grad_at_mode, const double* w, int n_p, const double* txyt,
                       const double* Xp, int p, const double* beta, double lik_sigma, double lik_lambda, int pred_m_v,
                       int n_samples, uint64_t seed, double* mu_latent, double* var_latent, double* p_rain,
                       double* amount_mean, double* amount_median, double* samples) {
  return guarded([&] {
    if (!s || !grad_at_mode || !w || (n_p > 0 && (!txyt || !mu_latent || !var_latent || !p_rain || !amount_mean ||
                                                  !amount_median)))
      config_error("stgp_zcptn_predict: null argument");
    if (n_samples < 2) config_error("zcptn_predict: need at least two samples for scoring");
    if (!(lik_sigma > 0.0) || !std::isfinite(lik_sigma)) config_error("LikelihoodParams: sigma must be > 0");
    if (!(lik_lambda > 0.0) || !std::isfinite(lik_lambda)) config_error("LikelihoodParams: lambda must be > 0");
    if (s->kind != STGP_FITC && s->policy != STGP_LATENT)
      numeric_error("LaplaceAlgebra: requires a latent-policy structure");
    if (n_p <= 0) return;
    laplace_release(s);
    zcptn_moments_dev(s, grad_at_mode, w, n_p, txyt, pred_m_v, mu_latent, var_latent);
    laplace_release(s);
    for (int q = 0; q < n_p; ++q) {
      double off = 0.0;
      if (p > 0 && Xp && beta)
        for (int j = 0; j < p; ++j) off += Xp[static_cast<size_t>(q) + static_cast<size_t>(j) * n_p] * beta[j];
      const double mu = off + mu_latent[q];
      const double var = var_latent[q];
      mu_latent[q] = mu;
      const double s_tot = std::sqrt(lik_sigma * lik_sigma + var);
      p_rain[q] = 1.0 - 0.5 * std::erfc((mu / s_tot) / 1.4142135623730951);
      std::mt19937_64 rng(mix_seed(seed, static_cast<uint64_t>(q)));
      std::normal_distribution<double> gauss(0.0, 1.0);
      const double sd = std::sqrt(var);
      double acc = 0.0;
      std::vector<double> draws(static_cast<size_t>(n_samples));
      for (int k = 0; k < n_samples; ++k) {
        const double latent = mu + sd * gauss(rng);
        const double zval = latent + lik_sigma * gauss(rng);
        const double amount = zval <= 0.0 ? 0.0 : std::pow(zval, lik_lambda);
        if (samples) samples[static_cast<size_t>(q) + static_cast<size_t>(k) * n_p] = amount;
        draws[static_cast<size_t>(k)] = amount;
        acc += amount;
      }
      amount_mean[q] = acc / n_samples;
      std::nth_element(draws.begin(), draws.begin() + n_samples / 2, draws.end());
      amount_median[q] = draws[static_cast<size_t>(n_samples) / 2];
    }
  });
}

}  // extern "C"

// Latent-policy likelihoods on the device: the Laplace algebra of
// approximations.cpp:1083-1375 (solves and log-determinants of Sigma^{-1} + W for diagonal W >= 0),
// the Gaussian latent-policy NLL (approximations.cpp:320-334), the ZC-PTN likelihood and Newton mode
// finding of laplace.cpp:25-203, and the ZC-PTN latent predictive moments (laplace.cpp:205-259).
//
// The reference factors the sparse Q + W (Q = B^T D^{-1} B) with a simplicial LDLT, a "desk scale"
// method.  Here Q is formed densely on the device (one thread per column over the CSC of
// B's pattern, rows in ascending order: the oracle's summation order) and Q + W is factored by the
// blocked DMMA Cholesky of dense.cu; the determinant and solves are the same quantities.  The dense
// form caps n at kMaxDense.  FITC and the VIF low-rank part are rewritten in the whitened basis
// W = L_m^{-1} U the structures already hold:
//   FITC  M_w = Sigma_m + U diag(dw) U^T = L_m (I + W diag(dw) W^T) L_m^T,
//   VIF   M_w = Sigma_m + U Q U^T - U Q S^{-1} Q U^T = L_m (I + W Q W^T - (Q W^T)^T S^{-1} (Q W^T)) L_m^T,
// so log|M_w| - log|Sigma_m| is the log-determinant of the bracket and the solves need only W.
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "dense.cuh"
#include "lowrank_common.cuh"
#include "../../include/stgp_b200.h"

namespace stgp {

constexpr int kMaxDense = 40000;

struct LaplaceDev {
  int n = 0, ldm = 0, M = 0, kind = 0;
  DevBuf<double> Q, S;          // n x n (Vecchia / VIF)
  DevBuf<double> QWt, Zw, Kw;   // VIF: Q W^T (n x ldm), S^{-1} Q W^T, bracket factor (ldm x ldm)
  DevBuf<double> scale, e1, l1; // FITC: 1 / (1 + w lam0), lam0 * scale, log(1 + w lam0)
  DevBuf<double> Ws;            // FITC: W diag(sqrt(dw)) (ldm x n)
  DevBuf<double> v1, v2, v3, vM, vM2;
  double logdet_sigma = 0.0, logdet_S = 0.0, logdet_K = 0.0, logdet_l1 = 0.0;
  bool prepared = false;
};

void laplace_release(stgp_structure* s) {
  delete s->lap;
  s->lap = nullptr;
}

namespace {

constexpr int kT = kLrThreads;

// Q(:, a) = sum over rows r referencing column a (ascending r) of B(r, a) B(r, :) / D_r
__global__ void form_q_kernel(int n, int m_v, const int32_t* __restrict__ nbr, const double* __restrict__ A,
                              const double* __restrict__ D, const int32_t* __restrict__ ptr,
                              const int32_t* __restrict__ erow, const int16_t* __restrict__ eslot, double* Q) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) {
    double* q = Q + static_cast<size_t>(a) * n;
    for (int p = ptr[a]; p < ptr[a + 1]; ++p) {
      const int r = erow[p], sl = eslot[p];
      const double ba = sl < 0 ? 1.0 : -A[static_cast<size_t>(r) * m_v + sl];
      const double dr = D[r];
      for (int b = 0; b < m_v; ++b) {
        const int j = nbr[static_cast<size_t>(r) * m_v + b];
        if (j < 0) continue;
        q[j] += ba * -A[static_cast<size_t>(r) * m_v + b] / dr;
      }
      q[r] += ba * 1.0 / dr;
    }
  }
}
__global__ void add_diag_kernel(int n, double* S, const double* w, double c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    S[static_cast<size_t>(i) * n + i] += w ? w[i] : c;
}
// FITC: scale = 1 / (1 + w lam0), e1 = lam0 scale, l1 = log(1 + w lam0), sq = sqrt(w scale)
__global__ void fitc_weights_kernel(int n, const double* w, double wc, const double* lam0, double* scale, double* e1,
                                    double* l1, double* sq) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double wi = w ? w[i] : wc;
    const double t = 1.0 + wi * lam0[i];
    const double sc = 1.0 / t;
    scale[i] = sc;
    e1[i] = lam0[i] * sc;
    l1[i] = log(t);
    sq[i] = sqrt(wi * sc);
  }
}
__global__ void mul_kernel(int n, const double* a, const double* b, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] * b[i];
}
__global__ void fma_vec_kernel(int n, const double* a, const double* x, const double* b, const double* y, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] * x[i] + b[i] * y[i];
}

// ---- ZC-PTN observation model (laplace.cpp:25-91) ----
constexpr double kLog2Pi = 1.8378770664093453;
__device__ double d_norm_pdf(double z) { return exp(-0.5 * z * z - 0.5 * kLog2Pi); }
__device__ double d_norm_cdf(double z) { return 0.5 * erfc(-z / 1.4142135623730951); }
__device__ double d_tail(double z) {
  const double z2 = z * z, z4 = z2 * z2;
  return 1.0 - 1.0 / z2 + 3.0 / z4 - 15.0 / (z4 * z2) + 105.0 / (z4 * z4) - 945.0 / (z4 * z4 * z2);
}
__device__ double d_log_norm_cdf(double z) {
  if (z > -8.0) return log(d_norm_cdf(z));
  return -0.5 * z * z - 0.5 * kLog2Pi - log(-z) + log(d_tail(z));
}
__device__ double d_inverse_mills(double z) {
  if (z > -8.0) return d_norm_pdf(z) / d_norm_cdf(z);
  return -z / d_tail(z);
}
__device__ double d_loglik(double y, double mu, double sigma, double lambda) {
  if (y == 0.0) return d_log_norm_cdf(-mu / sigma);
  const double g = pow(y, 1.0 / lambda);
  const double z = (g - mu) / sigma;
  return -0.5 * z * z - 0.5 * kLog2Pi - log(sigma) - log(lambda) - (1.0 - 1.0 / lambda) * log(y);
}
// g = d loglik / d mu, w = max(-d2, 0)
__global__ void zcptn_derivs_kernel(int n, const double* y, const double* off, const double* b, double sigma,
                                    double lambda, double* g, double* w) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double mu = off[i] + b[i];
    double d1, d2;
    if (y[i] == 0.0) {
      const double z = -mu / sigma;
      const double h = d_inverse_mills(z);
      d1 = -h / sigma;
      d2 = fmin((-z * h - h * h) / (sigma * sigma), 0.0);
    } else {
      d1 = (pow(y[i], 1.0 / lambda) - mu) / (sigma * sigma);
      d2 = -1.0 / (sigma * sigma);
    }
    g[i] = d1;
    w[i] = fmax(-d2, 0.0);
  }
}
// per-block partials of [sum loglik(b_try) - 0.5 a_try . b_try] with b_try = b + step (bn - b)
__global__ void psi_kernel(int n, const double* y, const double* off, const double* b, const double* bn,
                           const double* a, const double* an, double step, double sigma, double lambda, double* part) {
  __shared__ double red[kT];
  double s = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double bt = bn ? b[i] + step * (bn[i] - b[i]) : b[i];
    const double at = an ? a[i] + step * (an[i] - a[i]) : a[i];
    s += d_loglik(y[i], off[i] + bt, sigma, lambda) - 0.5 * (at * bt);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
// per-block max |g| and max |g - a|
__global__ void gap_kernel(int n, const double* g, const double* a, double* part) {
  __shared__ double r0[kT], r1[kT];
  double m0 = 0.0, m1 = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    m0 = fmax(m0, fabs(g[i]));
    m1 = fmax(m1, fabs(g[i] - a[i]));
  }
  r0[threadIdx.x] = m0;
  r1[threadIdx.x] = m1;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      r0[threadIdx.x] = fmax(r0[threadIdx.x], r0[threadIdx.x + o]);
      r1[threadIdx.x] = fmax(r1[threadIdx.x], r1[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = r0[0];
    part[2 * blockIdx.x + 1] = r1[0];
  }
}
// rhs = w b + g;  (after the solve) an = rhs - w bn
__global__ void newton_rhs_kernel(int n, const double* w, const double* b, const double* g, double* rhs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rhs[i] = w[i] * b[i] + g[i];
}
__global__ void newton_a_kernel(int n, const double* rhs, const double* w, const double* bn, double* an) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) an[i] = rhs[i] - w[i] * bn[i];
}
__global__ void step_kernel(int n, double step, double* b, const double* bn, double* a, const double* an) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    b[i] = b[i] + step * (bn[i] - b[i]);
    a[i] = a[i] + step * (an[i] - a[i]);
  }
}

}  // namespace

static LaplaceDev* lap_state(stgp_structure* s) {
  stgp_ctx* ctx = s->ds->ctx;
  if (s->lap) return s->lap;
  if (ctx->world > 1) config_error("Laplace algebra: run on an unsharded context (stgp_ctx_set_shard(ctx, 0, 1))");
  if (s->kind != STGP_FITC && s->policy != STGP_LATENT)
    numeric_error("LaplaceAlgebra: requires a latent-policy structure");
  if (s->kind != STGP_FITC && s->n > kMaxDense)
    config_error("Laplace algebra: the dense factorization of Q + W supports n <= 40000 (desk scale, SPEC.md:9)");
  auto L = std::make_unique<LaplaceDev>();
  L->n = s->n;
  L->kind = s->kind;
  L->M = s->kind == STGP_VECCHIA ? 0 : s->lr.M;
  L->ldm = s->kind == STGP_VECCHIA ? 0 : s->lr.ldm;
  const int n = s->n;
  cudaStream_t st = ctx->stream;
  if (s->kind != STGP_FITC) {
    ensure_csc(s);
    L->Q.ensure(static_cast<size_t>(n) * n);
    L->Q.zero(st);
    form_q_kernel<<<grid_for(n, 128), 128, 0, st>>>(n, s->m_v, s->nbr.get(), s->A.get(), s->D.get(),
                                                    s->csc_ptr.get(), s->csc_row.get(), s->csc_slot.get(),
                                                    L->Q.get());
    launched(ctx);
    L->logdet_sigma = dev_sum_log(ctx, s->D.get(), n, s->red);
    if (s->kind == STGP_VIF && L->M > 0) {  // Q W^T (n x ldm)
      L->QWt.ensure(static_cast<size_t>(n) * L->ldm);
      dev_gemm(ctx, false, true, n, L->ldm, n, 1.0, L->Q.get(), n, s->lr.W.get(), L->ldm, 0.0, L->QWt.get(), n);
    }
  }
  s->lap = L.release();
  return s->lap;
}

// prepare(w): w_dev (n) or the constant wc when w_dev is null
static void lap_prepare(stgp_structure* s, const double* w_dev, double wc) {
  LaplaceDev* L = lap_state(s);
  stgp_ctx* ctx = s->ds->ctx;
  cudaStream_t st = ctx->stream;
  const int n = L->n, ldm = L->ldm;
  if (L->kind == STGP_FITC) {
    LowRank& R = s->lr;
    L->scale.ensure(n);
    L->e1.ensure(n);
    L->l1.ensure(n);
    L->v3.ensure(n);
    fitc_weights_kernel<<<grid_for(n), kT, 0, st>>>(n, w_dev, wc, R.fitc_diag.get(), L->scale.get(), L->e1.get(),
                                                     L->l1.get(), L->v3.get());
    launched(ctx);
    L->logdet_l1 = dev_sum(ctx, L->l1.get(), n, s->red);
    L->Ws.ensure(static_cast<size_t>(ldm) * n);
    scale_cols(ctx, R.W.get(), ldm, n, L->v3.get(), false, L->Ws.get());
    L->Kw.ensure(static_cast<size_t>(ldm) * ldm);
    dev_gemm(ctx, false, true, ldm, ldm, n, 1.0, L->Ws.get(), ldm, L->Ws.get(), ldm, 0.0, L->Kw.get(), ldm);
    add_identity(ctx, L->Kw.get(), ldm);
    if (!dev_cholesky(ctx, L->Kw.get(), ldm, ldm)) numeric_error("FitcLaplace: core factorization failed");
    L->logdet_K = dev_logdet_chol(ctx, L->Kw.get(), ldm, ldm);
    L->prepared = true;
    return;
  }
  L->S.ensure(static_cast<size_t>(n) * n);
  STGP_CUDA(cudaMemcpyAsync(L->S.get(), L->Q.get(), sizeof(double) * n * n, cudaMemcpyDeviceToDevice, st));
  add_diag_kernel<<<grid_for(n), kT, 0, st>>>(n, L->S.get(), w_dev, wc);
  launched(ctx);
  if (!dev_cholesky(ctx, L->S.get(), n, n))
    numeric_error(L->kind == STGP_VECCHIA ? "VecchiaLaplace: factorization of Q + W failed"
                                          : "VifLaplace: factorization of Q + W failed");
  L->logdet_S = dev_logdet_chol(ctx, L->S.get(), n, n);
  if (L->kind == STGP_VIF && L->M > 0) {
    const LowRank& R = s->lr;
    L->Zw.ensure(static_cast<size_t>(n) * ldm);
    STGP_CUDA(cudaMemcpyAsync(L->Zw.get(), L->QWt.get(), sizeof(double) * n * ldm, cudaMemcpyDeviceToDevice, st));
    dev_trsm_left(ctx, L->S.get(), n, n, L->Zw.get(), n, ldm, false);
    dev_trsm_left(ctx, L->S.get(), n, n, L->Zw.get(), n, ldm, true);
    L->Kw.ensure(static_cast<size_t>(ldm) * ldm);
    dev_gemm(ctx, false, false, ldm, ldm, n, 1.0, R.W.get(), ldm, L->QWt.get(), n, 0.0, L->Kw.get(), ldm);
    dev_gemm(ctx, true, false, ldm, ldm, n, -1.0, L->QWt.get(), n, L->Zw.get(), n, 1.0, L->Kw.get(), ldm);
    add_identity(ctx, L->Kw.get(), ldm);
    if (!dev_cholesky(ctx, L->Kw.get(), ldm, ldm)) numeric_error("VifLaplace: core factorization failed");
    L->logdet_K = dev_logdet_chol(ctx, L->Kw.get(), ldm, ldm);
  }
  L->prepared = true;
}

static double lap_logdet(const LaplaceDev* L) {
  if (L->kind == STGP_FITC) return L->logdet_l1 + L->logdet_K;
  double v = L->logdet_S + L->logdet_sigma;
  if (L->kind == STGP_VIF && L->M > 0) v += L->logdet_K;
  return v;
}

// out = (Sigma^{-1} + W)^{-1} x (device vectors, n)
static void lap_solve(stgp_structure* s, const double* x, double* out) {
  LaplaceDev* L = s->lap;
  stgp_ctx* ctx = s->ds->ctx;
  cudaStream_t st = ctx->stream;
  const int n = L->n, ldm = L->ldm;
  L->vM.ensure(std::max(ldm, 1));
  if (L->kind == STGP_FITC) {
    L->v1.ensure(n);
    L->v2.ensure(n);
    mul_kernel<<<grid_for(n), kT, 0, st>>>(n, x, L->scale.get(), L->v1.get());
    launched(ctx);
    dev_gemv(ctx, false, ldm, n, 1.0, s->lr.W.get(), ldm, L->v1.get(), 0.0, L->vM.get());
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, L->vM.get(), ldm, 1, false);
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, L->vM.get(), ldm, 1, true);
    dev_gemv(ctx, true, ldm, n, 1.0, s->lr.W.get(), ldm, L->vM.get(), 0.0, L->v2.get());
    fma_vec_kernel<<<grid_for(n), kT, 0, st>>>(n, L->e1.get(), x, L->scale.get(), L->v2.get(), out);
    launched(ctx);
    return;
  }
  if (out != x) STGP_CUDA(cudaMemcpyAsync(out, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  dev_trsm_left(ctx, L->S.get(), n, n, out, n, 1, false);
  dev_trsm_left(ctx, L->S.get(), n, n, out, n, 1, true);
  if (L->kind == STGP_VIF && L->M > 0) {
    dev_gemv(ctx, true, n, ldm, 1.0, L->QWt.get(), n, out, 0.0, L->vM.get());  // (Q W^T)^T s0
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, L->vM.get(), ldm, 1, false);
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, L->vM.get(), ldm, 1, true);
    dev_gemv(ctx, false, n, ldm, 1.0, L->Zw.get(), n, L->vM.get(), 1.0, out);  // s0 += Zw K^{-1} (...)
  }
}

namespace {
__global__ void scale_rows_kernel(int n, long long ncols, const double* d, const double* X, double* out) {
  const long long total = static_cast<long long>(n) * ncols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    out[e] = X[e] * d[e % n];
}
__global__ void fitc_combine_kernel(int n, long long ncols, const double* e1, const double* X, const double* scale,
                                    const double* H, double* out) {
  const long long total = static_cast<long long>(n) * ncols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e % n;
    out[e] = e1[i] * X[e] + scale[i] * H[e];
  }
}
}  // namespace

void laplace_prepare_w(stgp_structure* s, const double* w_dev) {
  laplace_release(s);
  lap_prepare(s, w_dev, 0.0);
}

// out (n x ncols) = (Sigma^{-1} + W)^{-1} X after laplace_prepare_w
void laplace_solve_cols(stgp_structure* s, const double* X, long long ncols, double* out) {
  LaplaceDev* L = s->lap;
  stgp_ctx* ctx = s->ds->ctx;
  cudaStream_t st = ctx->stream;
  const int n = L->n, ldm = L->ldm;
  const int nc = static_cast<int>(ncols);
  if (L->kind == STGP_FITC) {
    DevBuf<double> T1(static_cast<size_t>(n) * nc), G(static_cast<size_t>(ldm) * nc), H(static_cast<size_t>(n) * nc);
    scale_rows_kernel<<<grid_for(static_cast<long long>(n) * nc), kT, 0, st>>>(n, nc, L->scale.get(), X, T1.get());
    launched(ctx);
    dev_gemm(ctx, false, false, ldm, nc, n, 1.0, s->lr.W.get(), ldm, T1.get(), n, 0.0, G.get(), ldm);
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, G.get(), ldm, nc, false);
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, G.get(), ldm, nc, true);
    dev_gemm(ctx, true, false, n, nc, ldm, 1.0, s->lr.W.get(), ldm, G.get(), ldm, 0.0, H.get(), n);
    fitc_combine_kernel<<<grid_for(static_cast<long long>(n) * nc), kT, 0, st>>>(n, nc, L->e1.get(), X, L->scale.get(),
                                                                                   H.get(), out);
    launched(ctx);
    return;
  }
  STGP_CUDA(cudaMemcpyAsync(out, X, sizeof(double) * n * nc, cudaMemcpyDeviceToDevice, st));
  dev_trsm_left(ctx, L->S.get(), n, n, out, n, nc, false);
  dev_trsm_left(ctx, L->S.get(), n, n, out, n, nc, true);
  if (L->kind == STGP_VIF && L->M > 0) {
    DevBuf<double> Q1(static_cast<size_t>(ldm) * nc);
    dev_gemm(ctx, true, false, ldm, nc, n, 1.0, L->QWt.get(), n, out, n, 0.0, Q1.get(), ldm);
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, Q1.get(), ldm, nc, false);
    dev_trsm_left(ctx, L->Kw.get(), ldm, ldm, Q1.get(), ldm, nc, true);
    dev_gemm(ctx, false, false, n, nc, ldm, 1.0, L->Zw.get(), n, Q1.get(), ldm, 1.0, out, n);
  }
}

// latent_policy_nll (approximations.cpp:320-334) on the structure's residual s->r
double latent_policy_nll_dev(stgp_structure* s) {
  const double sigma2 = s->th.sigma2;
  if (!(sigma2 > 0.0)) numeric_error("nll: the Gaussian path requires a positive nugget");
  stgp_ctx* ctx = s->ds->ctx;
  const int n = s->n;
  const double w = 1.0 / sigma2;
  lap_prepare(s, nullptr, w);
  LaplaceDev* L = s->lap;
  const double logdet = n * std::log(sigma2) + lap_logdet(L);
  L->v3.ensure(n);
  lap_solve(s, s->r.get(), L->v3.get());
  const double rr = dev_dot(ctx, s->r.get(), s->r.get(), n, s->red);
  const double rz = dev_dot(ctx, s->r.get(), L->v3.get(), n, s->red);
  const double quad = w * (rr - w * rz);
  return 0.5 * (logdet + quad + n * 1.8378770664093453);
}

namespace {
struct NewtonBufs {
  DevBuf<double> y, off, b, a, g, w, rhs, bn, an, part;
};

double psi_of(stgp_ctx* ctx, NewtonBufs& B, int n, const double* bn, const double* an, double step, double sigma,
              double lambda) {
  const int blocks = grid_for(n, kT, 256);
  B.part.ensure(static_cast<size_t>(2 * blocks));
  psi_kernel<<<blocks, kT, 0, ctx->stream>>>(n, B.y.get(), B.off.get(), B.b.get(), bn, B.a.get(), an, step, sigma,
                                             lambda, B.part.get());
  launched(ctx);
  std::vector<double> h(static_cast<size_t>(blocks));
  B.part.download(h.data(), h.size(), ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (double v : h) s += v;  // block order: deterministic
  return s;
}
bool gap_ok(stgp_ctx* ctx, NewtonBufs& B, int n) {
  const int blocks = grid_for(n, kT, 256);
  B.part.ensure(static_cast<size_t>(2 * blocks));
  gap_kernel<<<blocks, kT, 0, ctx->stream>>>(n, B.g.get(), B.a.get(), B.part.get());
  launched(ctx);
  std::vector<double> h(static_cast<size_t>(2 * blocks));
  B.part.download(h.data(), h.size(), ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  double mg = 0.0, md = 0.0;
  for (int k = 0; k < blocks; ++k) {
    mg = std::max(mg, h[static_cast<size_t>(2 * k)]);
    md = std::max(md, h[static_cast<size_t>(2 * k + 1)]);
  }
  return md < 1e-6 * std::max(1.0, mg);
}
}  // namespace

// laplace_marginal (laplace.cpp:115-203): Newton in (b, a = Sigma^{-1} b) with step halving on the
// penalised objective; returns -log marginal, leaves mode / grad_at_mode / w in the host arrays
double laplace_marginal_dev(stgp_structure* s, const double* y_host, const double* off_dev, double sigma,
                            double lambda, const double* warm_host, double* mode_out, double* a_out, double* w_out,
                            int* iters_out) {
  if (!(sigma > 0.0) || !std::isfinite(sigma)) config_error("LikelihoodParams: sigma must be > 0");
  if (!(lambda > 0.0) || !std::isfinite(lambda)) config_error("LikelihoodParams: lambda must be > 0");
  stgp_ctx* ctx = s->ds->ctx;
  cudaStream_t st = ctx->stream;
  const int n = s->n;
  for (int i = 0; i < n; ++i)
    if (y_host[i] < 0.0) data_error("zcptn_derivs: negative precipitation amount");
  lap_state(s);
  NewtonBufs B;
  for (DevBuf<double>* v : {&B.y, &B.off, &B.b, &B.a, &B.g, &B.w, &B.rhs, &B.bn, &B.an}) v->ensure(n);
  B.y.upload(y_host, n, st);
  if (off_dev) STGP_CUDA(cudaMemcpyAsync(B.off.get(), off_dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  else B.off.zero(st);
  bool warm_nonzero = false;
  if (warm_host)
    for (int i = 0; i < n && !warm_nonzero; ++i) warm_nonzero = warm_host[i] != 0.0;
  B.b.zero(st);
  B.a.zero(st);
  const int gb = grid_for(n);
  auto derivs = [&]() {
    zcptn_derivs_kernel<<<gb, kT, 0, st>>>(n, B.y.get(), B.off.get(), B.b.get(), sigma, lambda, B.g.get(), B.w.get());
    launched(ctx);
  };
  auto newton_target = [&]() {  // bn = (Sigma^{-1} + W)^{-1} (w b + g), an = rhs - w bn
    lap_prepare(s, B.w.get(), 0.0);
    newton_rhs_kernel<<<gb, kT, 0, st>>>(n, B.w.get(), B.b.get(), B.g.get(), B.rhs.get());
    launched(ctx);
    lap_solve(s, B.rhs.get(), B.bn.get());
    newton_a_kernel<<<gb, kT, 0, st>>>(n, B.rhs.get(), B.w.get(), B.bn.get(), B.an.get());
    launched(ctx);
  };
  if (warm_nonzero) {
    B.b.upload(warm_host, n, st);
    derivs();
    newton_target();
    STGP_CUDA(cudaMemcpyAsync(B.a.get(), B.an.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    STGP_CUDA(cudaMemcpyAsync(B.b.get(), B.bn.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  double psi = psi_of(ctx, B, n, nullptr, nullptr, 0.0, sigma, lambda);
  bool converged = false;
  int iter = 0;
  for (iter = 1; iter <= 100; ++iter) {
    derivs();
    if (gap_ok(ctx, B, n)) {
      converged = true;
      break;
    }
    newton_target();
    double step = 1.0;
    bool accepted = false;
    for (int h = 0; h < 30; ++h) {
      const double pt = psi_of(ctx, B, n, B.bn.get(), B.an.get(), step, sigma, lambda);
      if (pt >= psi - 1e-12 * std::abs(psi)) {
        step_kernel<<<gb, kT, 0, st>>>(n, step, B.b.get(), B.bn.get(), B.a.get(), B.an.get());
        launched(ctx);
        psi = pt;
        accepted = true;
        break;
      }
      step *= 0.5;
    }
    if (!accepted) break;
  }
  if (!converged) {
    derivs();
    converged = gap_ok(ctx, B, n);
    if (!converged) numeric_error("laplace_marginal: Newton did not converge in 100 iterations");
  }
  derivs();
  lap_prepare(s, B.w.get(), 0.0);
  const double lm = psi_of(ctx, B, n, nullptr, nullptr, 0.0, sigma, lambda) - 0.5 * lap_logdet(s->lap);
  if (mode_out) B.b.download(mode_out, n, st);
  if (a_out) B.a.download(a_out, n, st);
  if (w_out) B.w.download(w_out, n, st);
  STGP_CUDA(cudaStreamSynchronize(st));
  if (iters_out) *iters_out = iter;
  return -lm;
}

}  // namespace stgp

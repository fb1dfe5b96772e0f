// FITC in the whitened basis (approximations.cpp:238-275, 352-363, 495-571).
//
// With W = L_m^{-1} U and K = I + W Lambda^{-1} W^T (so M = L_m K L_m^T):
//   G1 = L_m^{-T} (K - I) L_m^T,  K2 = NL = L_m^{-T} K^{-1} W Lambda^{-1},
//   W2 = L_m^{-T} (I - K^{-1}) L_m^{-1},  P = L_m^{-T} W,
//   omega = L_m^{-T} [ K^{-1} W Lambda^{-1} - (W alpha) alpha^T - W diag(2 phi) ],
//   wsig  = L_m^{-T} [ -(I - K^{-1})/2 + (W alpha)(W alpha)^T / 2 + W diag(phi) W^T ] L_m^{-1},
// which removes the reference's n x M^2 GEMMs for G1 and W2.
#include "comm.hpp"
#include "dense.cuh"
#include "lowrank_common.cuh"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

namespace {

// fitc_diag = sigma1_2 - |W_i|^2 (clamped, approximations.cpp:253-263), lambda = diag + sigma2
__global__ void fitc_diag_kernel(int n, int M, int ldm, const double* W, double s1, double sigma2, double clamp_tol,
                                 double* diag, double* lambda, int* fail) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < n; i += nw) {
    double acc = 0.0;
    for (int j = lane; j < M; j += 32) {
      const double v = W[static_cast<size_t>(i) * ldm + j];
      acc = fma(v, v, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      double d = s1 - acc;
      if (d < 0.0) {
        if (d < -clamp_tol) atomicExch(fail, 1);
        d = 0.0;
      }
      diag[i] = d;
      const double l = d + sigma2;
      lambda[i] = l;
      if (l <= 0.0) atomicExch(fail, 2);
    }
  }
}

// per-column: out_i = |Hw_i|^2
__global__ void col_sqnorm_kernel(int n, int ldm, const double* A, double* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < n; i += nw) {
    double acc = 0.0;
    for (int j = lane; j < ldm; j += 32) {
      const double v = A[static_cast<size_t>(i) * ldm + j];
      acc = fma(v, v, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[i] = acc;
  }
}

// alpha_i = rl_i - t_i / lambda_i ; phi_i = 0.5 (1/lambda - |Hw_i|^2 / lambda^2 - alpha^2)
__global__ void fitc_alpha_phi_kernel(int n, const double* r, const double* lambda, const double* t, const double* hsq,
                                      double* alpha, double* phi) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double li = 1.0 / lambda[i];
    const double rl = r[i] * li;
    const double a = rl - li * t[i];
    alpha[i] = a;
    const double ds = li - hsq[i] * li * li;
    phi[i] = 0.5 * (ds - a * a);
  }
}

// omega'(:, i) = KW(:, i) / lambda_i - walpha * alpha_i - 2 phi_i W(:, i)   (in place into KW)
__global__ void fitc_omega_kernel(long long total, int ldm, const double* lambda, const double* alpha, const double* phi,
                                  const double* walpha, const double* W, double* KW) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / ldm;
    const int j = static_cast<int>(e % ldm);
    KW[e] = KW[e] / lambda[i] - walpha[j] * alpha[i] - 2.0 * phi[i] * W[e];
  }
}

// wsig' = -(I - Kinv)/2 + wa wa^T / 2 + S   (S = W diag(phi) W^T)
__global__ void fitc_wsig_kernel(int M, int ldm, const double* Kinv, const double* wa, const double* S, double* out) {
  const long long total = static_cast<long long>(ldm) * ldm;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e % ldm), c = static_cast<int>(e / ldm);
    double v = 0.0;
    if (r < M && c < M) v = -0.5 * ((r == c ? 1.0 : 0.0) - Kinv[e]) + 0.5 * wa[r] * wa[c] + S[e];
    out[e] = v;
  }
}

}  // namespace

void fitc_build(stgp_structure* s) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  prepare_tables(s);
  build_basis(s);
  build_cross(s, 0, s->n, false);
  const int n = s->n, ldm = L.ldm;
  L.fitc_diag.ensure(n);
  L.lambda.ensure(n);
  DevBuf<int> fail(1);
  fail.zero(ctx->stream);
  fitc_diag_kernel<<<grid_for(static_cast<long long>(n) * 32), 256, 0, ctx->stream>>>(
      n, L.M, ldm, L.W.get(), s->th.sigma1_2, s->th.sigma2, 1e-10 * std::max(1.0, s->th.sigma1_2), L.fitc_diag.get(),
      L.lambda.get(), fail.get());
  launched(ctx);
  int f = 0;
  fail.download(&f, 1, ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (f == 1) numeric_error("build_fitc: diagonal correction went negative");
  if (f == 2) numeric_error("build_fitc: zero observation diagonal; a positive nugget is required");
  // K = I + W Lambda^{-1} W^T
  const size_t total = static_cast<size_t>(ldm) * n;
  L.work1.ensure(total);
  scale_cols(ctx, L.W.get(), ldm, n, L.lambda.get(), true, L.work1.get());
  L.Mc.ensure(static_cast<size_t>(ldm) * ldm);
  set_identity(ctx, L.Mc.get(), ldm);
  dev_syrk(ctx, ldm, n, 1.0, L.work1.get(), ldm, 1.0, L.Mc.get(), ldm);
  dev_symmetrize_lower(ctx, L.Mc.get(), ldm, ldm);
  L.Kfull.ensure(static_cast<size_t>(ldm) * ldm);
  STGP_CUDA(cudaMemcpyAsync(L.Kfull.get(), L.Mc.get(), sizeof(double) * ldm * ldm, cudaMemcpyDeviceToDevice,
                            ctx->stream));
  if (!dev_cholesky(ctx, L.Mc.get(), ldm, ldm)) numeric_error("build_fitc: Woodbury core factorization failed");
  L.logdet_M = dev_logdet_chol(ctx, L.Mc.get(), ldm, ldm);
  s->built = true;
}

// shared prefix of NLL and gradient: rl, v = W rl, K^{-1} v, t = W^T K^{-1} W rl
static double fitc_core(stgp_structure* s, DevBuf<double>& rl, DevBuf<double>& kv, DevBuf<double>& t) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, ldm = L.ldm;
  rl.ensure(n);
  div_vec(ctx, n, s->r.get(), L.lambda.get(), rl.get());
  kv.ensure(ldm);
  dev_gemv(ctx, false, ldm, n, 1.0, L.W.get(), ldm, rl.get(), 0.0, kv.get());
  DevBuf<double> half(ldm);
  STGP_CUDA(cudaMemcpyAsync(half.get(), kv.get(), sizeof(double) * ldm, cudaMemcpyDeviceToDevice, ctx->stream));
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, half.get(), ldm, 1, false);
  const double vKv = dev_dot(ctx, half.get(), half.get(), ldm, s->red);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv.get(), ldm, 1, false);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv.get(), ldm, 1, true);
  t.ensure(n);
  dev_gemv(ctx, true, ldm, n, 1.0, L.W.get(), ldm, kv.get(), 0.0, t.get());
  const double rrl = dev_dot(ctx, s->r.get(), rl.get(), n, s->red);
  const double logl = dev_sum_log(ctx, L.lambda.get(), n, s->red);
  return 0.5 * (logl + L.logdet_M + rrl - vKv + nll_const(n));
}

double fitc_nll(stgp_structure* s) {
  DevBuf<double> rl, kv, t;
  return fitc_core(s, rl, kv, t);
}

void fitc_nll_grad(stgp_structure* s, double* nll, double* grad) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, M = L.M, ldm = L.ldm;
  cudaStream_t st = ctx->stream;
  DevBuf<double> rl, kv, t;
  const double v = fitc_core(s, rl, kv, t);
  if (nll) *nll = v;
  // Hw = L_K^{-1} W (|Hw_i|^2 -> diag of Sigma~^{-1}), KW = K^{-1} W
  const size_t total = static_cast<size_t>(ldm) * n;
  L.work1.ensure(total);
  STGP_CUDA(cudaMemcpyAsync(L.work1.get(), L.W.get(), sizeof(double) * total, cudaMemcpyDeviceToDevice, st));
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, L.work1.get(), ldm, n, false);
  DevBuf<double> hsq(n), alpha(n), phi(n), wa(ldm);
  col_sqnorm_kernel<<<grid_for(static_cast<long long>(n) * 32), 256, 0, st>>>(n, ldm, L.work1.get(), hsq.get());
  launched(ctx);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, L.work1.get(), ldm, n, true);
  fitc_alpha_phi_kernel<<<grid_for(n), 256, 0, st>>>(n, s->r.get(), L.lambda.get(), t.get(), hsq.get(), alpha.get(),
                                                     phi.get());
  launched(ctx);
  dev_gemv(ctx, false, ldm, n, 1.0, L.W.get(), ldm, alpha.get(), 0.0, wa.get());
  // S = W diag(phi) W^T ; wsig'
  L.work2.ensure(total);
  scale_cols(ctx, L.W.get(), ldm, n, phi.get(), false, L.work2.get());
  DevBuf<double> S(static_cast<size_t>(ldm) * ldm), Kinv(static_cast<size_t>(ldm) * ldm), Ws(static_cast<size_t>(ldm) * ldm);
  dev_gemm(ctx, false, true, ldm, ldm, n, 1.0, L.W.get(), ldm, L.work2.get(), ldm, 0.0, S.get(), ldm);
  set_identity(ctx, Kinv.get(), ldm);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, Kinv.get(), ldm, ldm, false);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, Kinv.get(), ldm, ldm, true);
  fitc_wsig_kernel<<<grid_for(static_cast<long long>(ldm) * ldm), 256, 0, st>>>(M, ldm, Kinv.get(), wa.get(), S.get(),
                                                                                Ws.get());
  launched(ctx);
  transform_wsig(ctx, L.Lm.get(), ldm, Ws.get());
  // omega' (in place of KW), omega = L_m^{-T} omega'
  fitc_omega_kernel<<<grid_for(static_cast<long long>(total)), 256, 0, st>>>(static_cast<long long>(total), ldm,
                                                                             L.lambda.get(), alpha.get(), phi.get(),
                                                                             wa.get(), L.W.get(), L.work1.get());
  launched(ctx);
  dev_trsm_left(ctx, L.Lm.get(), ldm, ldm, L.work1.get(), ldm, n, true);
  for (int q = 0; q < 7; ++q) grad[q] = 0.0;
  Reducer rr;
  const double phisum = dev_sum(ctx, phi.get(), n, rr);
  grad[0] += phisum;
  grad[1] += phisum;
  std::vector<double> gu = upair_grad(s, L.work1.get());
  std::vector<double> gs = sigma_pair_grad(s, Ws.get());
  for (int q = 0; q < 6; ++q) grad[1 + q] += gu[q] + gs[q];
}

}  // namespace stgp

// FITC in the whitened basis (approximations.cpp:238-275, 352-363, 495-571).
//
// With W = L_m^{-1} U and K = I + W Lambda^{-1} W^T (so M = L_m K L_m^T):
//   G1 = L_m^{-T} (K - I) L_m^T,  K2 = NL = L_m^{-T} K^{-1} W Lambda^{-1},
//   W2 = L_m^{-T} (I - K^{-1}) L_m^{-1},  P = L_m^{-T} W,
//   omega = L_m^{-T} [ K^{-1} W Lambda^{-1} - (W alpha) alpha^T - W diag(2 phi) ],
//   wsig  = L_m^{-T} [ -(I - K^{-1})/2 + (W alpha)(W alpha)^T / 2 + W diag(phi) W^T ] L_m^{-1},
// which removes the reference's n x M^2 GEMMs for G1 and W2.
#include <algorithm>
#include <cstdlib>

#include "comm.hpp"
#include "dense.cuh"
#include "lowrank_common.cuh"
#include "ozaki.cuh"
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
        if (d < -clamp_tol) atomicOr(fail, 1);
        d = 0.0;
      }
      diag[i] = d;
      const double l = d + sigma2;
      lambda[i] = l;
      if (l <= 0.0) atomicOr(fail, 2);
    }
  }
}

// per-column: out_i = A_i . B_i  (|L_K^{-1} W_i|^2 = W_i . (K^{-1} W)_i)
__global__ void col_dot_kernel(int n, int ldm, const double* A, const double* B, double* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = gw; i < n; i += nw) {
    double acc = 0.0;
    for (int j = lane; j < ldm; j += 32)
      acc = fma(A[static_cast<size_t>(i) * ldm + j], B[static_cast<size_t>(i) * ldm + j], acc);
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
// a block per column i (no 64-bit index division per element), two rows j per thread and step
__global__ void fitc_omega_kernel(long long ncols, int ldm, const double* lambda, const double* alpha, const double* phi,
                                  const double* walpha, const double* W, double* KW) {
  for (long long i = blockIdx.x; i < ncols; i += gridDim.x) {
    const double lam = lambda[i], al = alpha[i], ph2 = 2.0 * phi[i];
    const double2* w2 = reinterpret_cast<const double2*>(W + i * ldm);
    double2* k2 = reinterpret_cast<double2*>(KW + i * ldm);
    for (int j2 = threadIdx.x; j2 < ldm / 2; j2 += blockDim.x) {
      const double2 w = w2[j2];
      double2 k = k2[j2];
      k.x = k.x / lam - walpha[2 * j2] * al - ph2 * w.x;
      k.y = k.y / lam - walpha[2 * j2 + 1] * al - ph2 * w.y;
      k2[j2] = k;
    }
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
  {
    ProfRegion pr(ctx, "basis");
    build_basis(s);
  }
  const int rb = s->row_begin, re = s->row_end, ldm = L.ldm, n = s->n;
  build_cross(s, rb, re, false);
  L.fitc_diag.ensure(n);
  L.lambda.ensure(n);
  DevBuf<int> fail(1);
  fail.zero(ctx->stream);
  const size_t own = static_cast<size_t>(rb) * ldm;
  if (re > rb) {
    fitc_diag_kernel<<<grid_for(static_cast<long long>(re - rb) * 32), 256, 0, ctx->stream>>>(
        re - rb, L.M, ldm, L.W.get() + own, s->th.sigma1_2, s->th.sigma2, 1e-10 * std::max(1.0, s->th.sigma1_2),
        L.fitc_diag.get() + rb, L.lambda.get() + rb, fail.get());
    launched(ctx);
  }
  std::vector<double> f(2, 0.0);
  {
    int fi = 0;
    fail.download(&fi, 1, ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
    f[0] = (fi & 1) ? 1.0 : 0.0;
    f[1] = (fi & 2) ? 1.0 : 0.0;
  }
  allreduce_host(ctx, f);  // every rank raises the same error
  if (f[0] > 0.0) numeric_error("build_fitc: diagonal correction went negative");
  if (f[1] > 0.0) numeric_error("build_fitc: zero observation diagonal; a positive nugget is required");
  // K = I + sum_shards W Lambda^{-1} W^T
  const size_t total = static_cast<size_t>(ldm) * n;
  L.work1.ensure(total);
  L.Mc.ensure(static_cast<size_t>(ldm) * ldm);
  STGP_CUDA(cudaMemsetAsync(L.Mc.get(), 0, sizeof(double) * ldm * ldm, ctx->stream));
  ProfRegion prk(ctx, "K_gemm_chol");
  if (re > rb) {
    if (ozaki_for(ldm)) {  // W Lambda^{-1} W^T on the int8 tensor cores
      ozaki_syrk_keep(ctx, ldm, re - rb, L.W.get() + own, ldm, L.lambda.get() + rb, L.Mc.get(), ldm, s->uid);
    } else {
      scale_cols(ctx, L.W.get() + own, ldm, re - rb, L.lambda.get() + rb, true, L.work1.get() + own);
      dev_syrk_blocked(ctx, ldm, re - rb, 1.0, L.work1.get() + own, ldm, L.Mc.get(), ldm, 4);
    }
  }
  allreduce_sum(ctx, L.Mc.get(), static_cast<size_t>(ldm) * ldm);
  add_identity(ctx, L.Mc.get(), ldm);
  L.Kfull.ensure(static_cast<size_t>(ldm) * ldm);
  STGP_CUDA(cudaMemcpyAsync(L.Kfull.get(), L.Mc.get(), sizeof(double) * ldm * ldm, cudaMemcpyDeviceToDevice,
                            ctx->stream));
  if (!dev_cholesky(ctx, L.Mc.get(), ldm, ldm)) numeric_error("build_fitc: Woodbury core factorization failed");
  L.logdet_M = dev_logdet_chol(ctx, L.Mc.get(), ldm, ldm);
  s->built = true;
}

// shared prefix of NLL and gradient (own rows): rl, v = W rl (summed), kv = K^{-1} v, t = W^T kv
// W diag(phi) W^T from the tiles of one triangle, mirrored (STGP_FITC_SYM_S=0: all tiles, then the
// lower triangle copied up)
static bool sym_S() {
  static const bool on = [] {
    const char* e = std::getenv("STGP_FITC_SYM_S");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

static double fitc_core(stgp_structure* s, double*& rl, double*& kv, double*& t) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, ldm = L.ldm, rb = s->row_begin, re = s->row_end;
  const size_t own = static_cast<size_t>(rb) * ldm;
  rl = L.tmp("f_rl", n);
  kv = L.tmp("f_kv", ldm);
  t = L.tmp("f_t", n);
  double* half = L.tmp("f_half", ldm);
  STGP_CUDA(cudaMemsetAsync(kv, 0, sizeof(double) * ldm, ctx->stream));
  std::vector<double> parts(2, 0.0);
  if (re > rb) {
    div_vec(ctx, re - rb, s->r.get() + rb, L.lambda.get() + rb, rl + rb);
    dev_gemv(ctx, false, ldm, re - rb, 1.0, L.W.get() + own, ldm, rl + rb, 0.0, kv);
    parts[0] = dev_dot(ctx, s->r.get() + rb, rl + rb, re - rb, s->red);
    parts[1] = dev_sum_log(ctx, L.lambda.get() + rb, re - rb, s->red);
  }
  allreduce_sum(ctx, kv, ldm);
  allreduce_host(ctx, parts);
  STGP_CUDA(cudaMemcpyAsync(half, kv, sizeof(double) * ldm, cudaMemcpyDeviceToDevice, ctx->stream));
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, half, ldm, 1, false);
  const double vKv = dev_dot(ctx, half, half, ldm, s->red);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, false);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, true);
  if (re > rb) dev_gemv(ctx, true, ldm, re - rb, 1.0, L.W.get() + own, ldm, kv, 0.0, t + rb);
  return 0.5 * (parts[1] + L.logdet_M + parts[0] - vKv + nll_const(n));
}

double fitc_nll(stgp_structure* s) {
  double *rl, *kv, *t;
  return fitc_core(s, rl, kv, t);
}

void fitc_nll_grad(stgp_structure* s, double* nll, double* grad) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, M = L.M, ldm = L.ldm, rb = s->row_begin, re = s->row_end, nown = re - rb;
  const size_t own = static_cast<size_t>(rb) * ldm, mm = static_cast<size_t>(ldm) * ldm;
  cudaStream_t st = ctx->stream;
  double *rl, *kv, *t;
  const double v = fitc_core(s, rl, kv, t);
  if (nll) *nll = v;
  double *hsq = L.tmp("f_hsq", n), *alpha = L.tmp("f_alpha", n), *phi = L.tmp("f_phi", n), *wa = L.tmp("f_wa", ldm),
         *S = L.tmp("f_S", mm), *Ws = L.tmp("f_Ws", mm);
  const size_t total = static_cast<size_t>(ldm) * n;
  L.work1.ensure(total);
  L.work2.ensure(total);
  STGP_CUDA(cudaMemsetAsync(wa, 0, sizeof(double) * ldm, st));
  STGP_CUDA(cudaMemsetAsync(S, 0, sizeof(double) * mm, st));
  std::vector<double> phisum(1, 0.0);
  // explicit K^{-1} (M^3): KW = K^{-1} W is one GEMM, and |L_K^{-1} W_i|^2 = W_i . KW_i
  L.Kinv.ensure(mm);
  dev_chol_inverse(ctx, L.Mc.get(), ldm, ldm, L.Kinv.get());
  if (nown > 0) {
    {
      ProfRegion pr(ctx, "f_KW_gemm");
      if (ozaki_for(ldm))  // K^{-1} symmetric: KW_i = K^{-1} W_i row by row
        ozaki_gemm_rows(ctx, nown, ldm, ldm, L.W.get() + own, ldm, L.Kinv.get(), ldm, L.work1.get() + own, ldm);
      else
        dev_gemm(ctx, false, false, ldm, nown, ldm, 1.0, L.Kinv.get(), ldm, L.W.get() + own, ldm, 0.0,
                 L.work1.get() + own, ldm);
      col_dot_kernel<<<grid_for(static_cast<long long>(nown) * 32), 256, 0, st>>>(nown, ldm, L.W.get() + own,
                                                                                 L.work1.get() + own, hsq + rb);
      launched(ctx);
      fitc_alpha_phi_kernel<<<grid_for(nown), 256, 0, st>>>(nown, s->r.get() + rb, L.lambda.get() + rb, t + rb,
                                                            hsq + rb, alpha + rb, phi + rb);
      launched(ctx);
      dev_gemv(ctx, false, ldm, nown, 1.0, L.W.get() + own, ldm, alpha + rb, 0.0, wa);
    }
    // S = W diag(phi) W^T (symmetric: lower blocks only)
    ProfRegion prs(ctx, "f_S_gemm");
    if (ozaki_for(ldm)) {  // S(i, j) = sum_r W(i, r) phi_r W(j, r); mirrored lower triangle
      // (W Lambda^{-1/2}) digits kept from K: S = (W Lambda^{-1/2}) (W diag(phi Lambda^{1/2}))^T, the column
      // factors applied by the slicer
      if (!ozaki_gemm_kept(ctx, ldm, nown, L.W.get() + own, ldm, L.lambda.get() + rb, S, ldm, s->uid, sym_S(),
                           phi + rb)) {
        scale_cols(ctx, L.W.get() + own, ldm, nown, phi + rb, false, L.work2.get() + own);
        ozaki_gemm_cols(ctx, ldm, nown, L.work2.get() + own, ldm, L.W.get() + own, ldm, S, ldm);
      }
      dev_symmetrize_lower(ctx, S, ldm, ldm);
    } else {
      scale_cols(ctx, L.W.get() + own, ldm, nown, phi + rb, false, L.work2.get() + own);
      dev_gemm_sym_blocked(ctx, ldm, nown, 1.0, L.W.get() + own, ldm, L.work2.get() + own, ldm, S, ldm, 4);
    }
    Reducer rr;
    phisum[0] = dev_sum(ctx, phi + rb, nown, rr);
  }
  allreduce_sum(ctx, wa, ldm);
  allreduce_sum(ctx, S, mm);
  allreduce_host(ctx, phisum);
  fitc_wsig_kernel<<<grid_for(static_cast<long long>(mm)), 256, 0, st>>>(M, ldm, L.Kinv.get(), wa, S, Ws);
  launched(ctx);
  transform_wsig(ctx, L.Lminv.get(), ldm, Ws);
  std::vector<double> g(7, 0.0);
  if (nown > 0) {
    // omega' (in place of KW), omega = L_m^{-T} omega'
    fitc_omega_kernel<<<static_cast<int>(std::min<long long>(nown, ctx->num_sms * 16LL)), 256, 0, st>>>(
        nown, ldm, L.lambda.get() + rb, alpha + rb, phi + rb, wa, L.W.get() + own, L.work1.get() + own);
    launched(ctx);
    ProfRegion pr(ctx, "f_omega_trmm_upair");
    lr_trmm(ctx, L.Lminv.get(), ldm, L.work1.get() + own, nown, true, L.work2.get() + own);
    std::vector<double> gu = upair_grad(s, L.work2.get(), rb, re);
    for (int q = 0; q < 6; ++q) g[1 + q] += gu[q];
  }
  if (ctx->rank == 0) {
    std::vector<double> gs = sigma_pair_grad(s, Ws);
    for (int q = 0; q < 6; ++q) g[1 + q] += gs[q];
  }
  allreduce_host(ctx, g);
  for (int q = 0; q < 7; ++q) grad[q] = g[q];
  grad[0] += phisum[0];
  grad[1] += phisum[0];
}

}  // namespace stgp

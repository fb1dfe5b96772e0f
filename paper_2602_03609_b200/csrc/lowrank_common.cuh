// Host helpers shared by the low-rank translation units (lowrank.cu, fitc.cu, predict.cu).
#pragma once
#include <vector>

#include "structure.hpp"

namespace stgp {

constexpr int kLrThreads = 256;
inline int grid_for(long long work, int per = kLrThreads, int cap = 148 * 32) {
  return static_cast<int>(std::max<long long>(1, std::min<long long>((work + per - 1) / per, cap)));
}
inline void launched(stgp_ctx* ctx) {
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
}

void build_basis(stgp_structure* s);                               // Sigma_m Cholesky + jitter ladder
void build_cross(stgp_structure* s, int c0, int c1, bool keep_U);  // U, W = L_m^{-1} U
void ensure_csc(stgp_structure* s);
void b_apply(stgp_structure* s, const double* v, double* out);     // B v
void bt_apply(stgp_structure* s, const double* v, double* out);    // B^T v
void scale_cols(stgp_ctx* ctx, const double* in, int ldm, long long ncols, const double* s, bool rsqrt_of, double* out);
void set_identity(stgp_ctx* ctx, double* A, int ld);
void div_vec(stgp_ctx* ctx, int n, const double* x, const double* d, double* y);
void vsub(stgp_ctx* ctx, long long n, const double* a, const double* b, double* out);  // a - b
void vadd(stgp_ctx* ctx, long long n, const double* a, const double* b, double* out);  // a + b
void sigma_inv_apply_dev(stgp_structure* s, const double* v, double* out);
void gls_beta_device(stgp_structure* s, const double* y_host, const double* X_host, int p, double* beta_out);
double dev_dot(stgp_ctx* ctx, const double* a, const double* b, long long n, Reducer& red);
double dev_sum(stgp_ctx* ctx, const double* v, long long n, Reducer& red);
double dev_sum_log(stgp_ctx* ctx, const double* v, long long n, Reducer& red);
// wsig = L_m^{-T} wsig' L_m^{-1} in place
void transform_wsig(stgp_ctx* ctx, const double* Lminv, int ldm, double* Ws);
// C = op(L_m^{-1}) B over ncols columns (ldm): the n x M^2 triangular products W = L_m^{-1} U and
// omega = L_m^{-T} omega' -- the tcgen05 Ozaki rows form at M >= STGP_OZAKI_MIN_M, else the DMMA TRMM
void lr_trmm(stgp_ctx* ctx, const double* Lminv, int ldm, const double* B, long long ncols, bool transpose, double* C);
// sum_{j,i} Om(j,i) dk(z_j, p_i) and the Sigma_m-pair sum (6 components each)
std::vector<double> upair_grad(stgp_structure* s, const double* Om, int c0, int c1);
void add_identity(stgp_ctx* ctx, double* A, int ld);
void compute_halo(stgp_structure* s);  // col_begin = min neighbour index over this shard's rows
std::vector<double> sigma_pair_grad(stgp_structure* s, const double* Ws);
double fitc_nll(stgp_structure* s);
void fitc_nll_grad(stgp_structure* s, double* nll, double* grad);

}  // namespace stgp

/*
 * stgp CPU oracle — C ABI.
 *
 * TEST INFRASTRUCTURE ONLY.  This library restates the reference's hot path
 * (/root/reference/proj: covariance.cpp, neighbors.cpp, inducing.cpp,
 * dataset.cpp:81-114, approximations.cpp:26-1080) on the CPU so that the CUDA
 * engine can be checked against it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * (paper_2602_03609_b200/libstgp_b200.so) never links or calls it.
 *
 * Parity pinning: the reference cannot be built here (Eigen3 and vendor/ are
 * absent), so the restatement is pinned against the
 * reference's own known-answer tests (tests/test_oracle_pinning.py).
 *
 * Reduction-order convention (documented in DESIGN.md §3): every dot-like
 * accumulation whose bits feed a bit-exact output (Σ_m Cholesky, whitening
 * W = L⁻¹U, w_i·w_j in d_r) is a sequential fused multiply-add chain in
 * increasing index order.  Eigen's own order is not recoverable here.
 *
 * Return codes: 0 ok, 2 ConfigError, 3 DataError, 4 NumericError, 1 other.
 */
#ifndef STGP_ORACLE_H
#define STGP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double sigma2, sigma1_2, a, c, alpha, nu, beta, delta;
} orc_params;

/* One model description; all arrays are host arrays in the ordered index
 * space.  kind: 0 Vecchia, 1 FITC, 2 VIF.  policy: 0 latent, 1 observation.
 * nbr is an n*m_v ELL array (ascending indices, -1 padded). */
typedef struct {
  int kind;
  int policy;
  int n;
  const double *x, *y, *t;
  const int32_t* nbr;
  int m_v;
  int M;
  const double *zx, *zy, *zt;
  orc_params theta;
} orc_model;

const char* orc_last_error(void);
double orc_exp(double x);
void orc_exp_array(long n, const double* x, double* out);
uint64_t orc_mix_seed(uint64_t seed, uint64_t stream);
double orc_kernel_eval(const orc_params* p, double h, double u);
int orc_kernel_grad(const orc_params* p, double h, double u, double* g6);
int orc_effective_ranges(const orc_params* p, double* time_range, double* space_range);

int orc_order_observations(int n, const double* t, uint64_t seed, int32_t* perm);

double orc_dc_pair(const orc_params* p, double xa, double ya, double ta, double xb,
                   double yb, double tb);
int orc_dc_neighbors(int n, const double* x, const double* y, const double* t,
                     const orc_params* p, int m_v, int32_t* out, double* dist);
int orc_dr_neighbors(int n, const double* x, const double* y, const double* t,
                     const orc_params* p, int M, const double* zx, const double* zy,
                     const double* zt, int m_v, int32_t* out, double* dist,
                     double* W_out, double* resid_out);
/* residual_neighbors for chosen query rows (rows == NULL: 0..nq-1) with certified exact pruning; rows must
 * be time ordered; out / dist are nq x m_v; by_dist != 0 lists each row's indices in (distance, index)
 * order instead of ascending */
int orc_dr_neighbors_rows(int n, const double* x, const double* y, const double* t, const orc_params* p, int M,
                          const double* zx, const double* zy, const double* zt, int m_v, int nq,
                          const int32_t* rows, int32_t* out, double* dist, int by_dist);
int orc_euclid_neighbors(int n, const double* x, const double* y, const double* t,
                         int m_v, double space_scale, double time_scale, int32_t* out);
/* brute-force cover-tree emulation over query subset [q0,q1) only (CPU baseline) */
int orc_dc_neighbors_range(int n, const double* x, const double* y, const double* t,
                           const orc_params* p, int m_v, int q0, int q1, int32_t* out);

int orc_kmeanspp(const double* pts_colmajor, int n, int d, int k, uint64_t seed,
                 double* centers_colmajor);
int orc_sts_kmeanspp(int n, const double* x, const double* y, const double* t, int m,
                     uint64_t seed, int* m_s, int* m_t, double* out_xyt, int cap);
int orc_joint_kmeanspp(int n, const double* x, const double* y, const double* t, int m,
                       double space_scale, double time_scale, uint64_t seed, int* k_out,
                       double* out_xyt, int cap);
int orc_inducing_logdet(int M, const double* zx, const double* zy, const double* zt,
                        const orc_params* p, int with_table_n, const double* data_t,
                        double* logdet);

/* approximations (approximations.cpp) */
int orc_build_rows(const orc_model* m, double* D_out, double* A_out);
int orc_nll(const orc_model* m, const double* yv, int p, const double* X,
            const double* beta, double* out);
int orc_nll_grad(const orc_model* m, const double* yv, int p, const double* X,
                 const double* beta, double* grad7);
/* nll_grad plus, per component, the sum over rows of |row contribution| (the tolerance yardstick) */
int orc_nll_grad_scale(const orc_model* m, const double* yv, int p, const double* X, const double* beta,
                       double* grad7, double* scale7);
int orc_zcptn(double y, double mu, double sigma, double lambda, double* out3);
void orc_normal_tail(double z, double* out3);
/* laplace_marginal (laplace.cpp:115-203) with the ZC-PTN likelihood: negative log-marginal and the state
 * at the mode (mode, grad_at_mode, w: n each, may be NULL); warm may be NULL */
int orc_laplace_marginal(const orc_model* m, const double* yv, int p, const double* X, const double* beta,
                         double lik_sigma, double lik_lambda, const double* warm, double* nll_out, double* mode,
                         double* grad_at_mode, double* w_out, int* iterations);
/* zcptn_predict (laplace.cpp:205-259); samples n_p x n_samples column-major (may be NULL); var_scale (may
 * be NULL): |k_pp| + |k'Wk| + |(Wk)'(Sigma^-1 + W)^-1 (Wk)|, the magnitude the variance cancels from */
int orc_zcptn_predict(const orc_model* m, const double* grad_at_mode, const double* w, int n_p, const double* qx,
                      const double* qy, const double* qt, const double* Xp, int p, const double* beta,
                      double lik_sigma, double lik_lambda, int pred_m_v, int n_samples, uint64_t seed,
                      double* mu_latent, double* var_latent, double* p_rain, double* amount_mean,
                      double* amount_median, double* samples, double* var_scale);
int orc_gls_beta(const orc_model* m, const double* yv, int p, const double* X,
                 double* beta_out);
int orc_predict(const orc_model* m, const double* yv, int p, const double* X,
                const double* beta, int n_p, const double* qx, const double* qy,
                const double* qt, const double* Xp, int pred_m_v, double* mu, double* var);
int orc_fitc_diag(const orc_model* m, double* fitc_diag);

/* DenseOracle (tests/oracles.cpp:24-112): long-double kernel, dense LLT */
int orc_dense_nll(int n, const double* x, const double* y, const double* t,
                  const orc_params* p, const double* yv, int pc, const double* X,
                  const double* beta, double* out);
int orc_dense_predict(int n, const double* x, const double* y, const double* t,
                      const orc_params* p, const double* yv, int n_p, const double* qx,
                      const double* qy, const double* qt, double* mu, double* var);

int orc_test_dataset(int kind, int n, uint64_t seed, int n_times, int p, double* x,
                     double* y, double* t, double* yv, double* X);

int orc_set_threads(int n);
/* 1 (default): exact lag-bound block pruning in the d_c scan; 0: plain brute force */
int orc_set_prune(int on);
/* BLAS timing mode: dense n x M^2 contractions through the OpenBLAS at path (scipy-bundled LP64, symbols
 * scipy_dgemm_ etc.) with the given thread count; path NULL or "" restores the sequential restatement */
int orc_set_blas(const char* path, int threads);

#ifdef __cplusplus
}
#endif
#endif

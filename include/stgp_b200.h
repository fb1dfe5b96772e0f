/*
 * stgp_b200 — C ABI of the B200-native engine for the data-parallel hot path of
 * arXiv 2602.03609 (Vecchia / FITC / VIF likelihood, gradient and prediction,
 * correlation-based neighbour search, space-time kMeans++ seeding).
 *
 * Every entry point replaces one reference C++ function (reference paths are
 * relative to /root/reference/proj); the C++ facade in include/stgp_b200.hpp
 * re-exposes them with the reference's names and exception types, and
 * INTEGRATION.md shows the binding a maintainer adds on the reference side.
 *
 * Conventions
 *  - All pointers named *_host are host memory; results are written to host
 *    memory.  Device memory never crosses the boundary.
 *  - Datasets are in the ordered index space of order_observations
 *    (dataset.cpp:81-114); stgp_order_observations computes that permutation.
 *  - Neighbour sets are n x m_v int32 row-major, ascending indices, -1 padded
 *    (NeighborSets.sets, neighbors.hpp:100-110).
 *  - Matrices (X, points) are column-major like Eigen's den_mat_t.
 *  - Return codes mirror the reference exception classes (types.hpp:26-38):
 *    0 ok, 2 ConfigError, 3 DataError, 4 NumericError, 1 internal/CUDA error.
 *    stgp_last_error() returns the calling thread's last message.
 *  - Calls are synchronous on the context's stream; objects belong to one
 *    context and must not be used from two threads at once.
 */
#ifndef STGP_B200_H
#define STGP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STGP_OK 0
#define STGP_ERR_INTERNAL 1
#define STGP_ERR_CONFIG 2
#define STGP_ERR_DATA 3
#define STGP_ERR_NUMERIC 4

/* approximation kinds and diagonal policies (approximations.hpp:31) */
#define STGP_VECCHIA 0
#define STGP_FITC 1
#define STGP_VIF 2
#define STGP_LATENT 0
#define STGP_OBSERVATION 1

/* NeighborSets::MetricKind (neighbors.hpp:101) */
#define STGP_METRIC_EUCLID 0
#define STGP_METRIC_DC 1
#define STGP_METRIC_DR 2

/* CovarianceParams (covariance.hpp:23-38), same field order */
typedef struct {
  double sigma2, sigma1_2, a, c, alpha, nu, beta, delta;
} stgp_params;

typedef struct stgp_ctx stgp_ctx;
typedef struct stgp_dataset stgp_dataset;
typedef struct stgp_neighbors stgp_neighbors;
typedef struct stgp_inducing stgp_inducing;
typedef struct stgp_structure stgp_structure;

const char* stgp_last_error(void);
int stgp_version(void);

/* ---- context: one CUDA device + stream (+ optional NCCL communicator) ---- */
int stgp_ctx_create(int device, stgp_ctx** out);
void stgp_ctx_destroy(stgp_ctx* ctx);
int stgp_ctx_synchronize(stgp_ctx* ctx);
/* Observation sharding for multi-GPU runs: this context owns rows
 * [n*rank/world, n*(rank+1)/world).  Partial sums are all-reduced through NCCL
 * when a communicator is attached, otherwise returned as this shard's partial. */
int stgp_ctx_set_shard(stgp_ctx* ctx, int rank, int world);
int stgp_nccl_unique_id(void* out128);
int stgp_ctx_init_nccl(stgp_ctx* ctx, const void* unique_id128, int rank, int world);
/* Sum all-reduce over host buffers supplied by the caller instead of NCCL
 * (in-process ranks on one device, test harnesses).  fn returns 0 on success. */
typedef int (*stgp_allreduce_fn)(void* user, double* buf, int64_t count);
int stgp_ctx_set_host_allreduce(stgp_ctx* ctx, stgp_allreduce_fn fn, void* user);
/* the context's cudaStream_t (for event timing by the caller) */
void* stgp_ctx_stream(stgp_ctx* ctx);
/* live per-kernel timing with CUDA events on the context stream (off by default):
 * region names are the kernel families ("rows", "knn", ...). */
int stgp_ctx_profile(stgp_ctx* ctx, int enable);
int stgp_ctx_profile_get(stgp_ctx* ctx, const char* region, double* total_ms, int64_t* count);
int stgp_ctx_profile_reset(stgp_ctx* ctx);
/* number of this library's kernels launched through ctx so far */
int64_t stgp_ctx_kernel_launches(const stgp_ctx* ctx);

/* ---- host ordering helper: order_observations (dataset.cpp:81-114) ---- */
int stgp_order_observations(int n, const double* t_host, uint64_t seed, int32_t* perm_out);
/* effective_ranges (covariance.cpp:231-254) */
int stgp_effective_ranges(const stgp_params* theta, double* time_range, double* space_range);
/* mix_seed (types.hpp:65-70) */
uint64_t stgp_mix_seed(uint64_t seed, uint64_t stream);

/* ---- dataset: device-resident SoA of ordered observations ---- */
int stgp_dataset_create(stgp_ctx* ctx, int n, const double* x_host, const double* y_host,
                        const double* t_host, stgp_dataset** out);
/* response and covariates kept resident on the device (used when a y_host
 * argument below is NULL).  X is n x p column-major. */
int stgp_dataset_set_response(stgp_dataset* ds, const double* resp_host, int p, const double* X_host);
void stgp_dataset_destroy(stgp_dataset* ds);

/* ---- neighbour selection (neighbors.hpp:112-125) ---- */
int stgp_euclidean_neighbors(stgp_dataset* ds, int m_v, double space_scale, double time_scale,
                             stgp_neighbors** out);
int stgp_correlation_neighbors(stgp_dataset* ds, const stgp_params* theta, int m_v,
                               stgp_neighbors** out);
int stgp_residual_neighbors(stgp_dataset* ds, const stgp_params* theta, const stgp_inducing* ind,
                            int m_v, stgp_neighbors** out);
/* caller-supplied sets (e.g. full conditioning); rows ascending, -1 padded */
int stgp_neighbors_from_host(stgp_dataset* ds, int m_v, const int32_t* idx_host, int metric_kind,
                             stgp_neighbors** out);
int stgp_neighbors_shape(const stgp_neighbors* nb, int* n, int* m_v, int* metric_kind);
/* indices (n*m_v) and, when the set came from a search, distances sorted
 * ascending per row (n*m_v, NaN padded); dist may be NULL */
int stgp_neighbors_download(const stgp_neighbors* nb, int32_t* idx_out, double* dist_out);
void stgp_neighbors_destroy(stgp_neighbors* nb);

/* ---- inducing points (inducing.hpp:22-75) ---- */
int stgp_inducing_create(stgp_ctx* ctx, int M, const double* xyt_host, stgp_inducing** out);
int stgp_sts_kmeanspp(stgp_dataset* ds, int m, uint64_t seed, stgp_inducing** out);
int stgp_joint_kmeanspp_inducing(stgp_dataset* ds, int m, double space_scale, double time_scale,
                                 uint64_t seed, stgp_inducing** out);
/* plain kmeanspp on an n x d column-major point matrix (inducing.cpp:46-115) */
int stgp_kmeanspp(stgp_ctx* ctx, const double* points_host, int n, int d, int k, uint64_t seed,
                  double* centers_out);
int stgp_inducing_size(const stgp_inducing* ind, int* M, int* m_s, int* m_t);
int stgp_inducing_download(const stgp_inducing* ind, double* xyt_out);
void stgp_inducing_destroy(stgp_inducing* ind);

/* ---- structures (approximations.hpp:89-100) ---- */
int stgp_build_vecchia(stgp_dataset* ds, const stgp_params* theta, const stgp_neighbors* nb,
                       int policy, stgp_structure** out);
int stgp_build_fitc(stgp_dataset* ds, const stgp_params* theta, const stgp_inducing* ind,
                    stgp_structure** out);
int stgp_build_vif(stgp_dataset* ds, const stgp_params* theta, const stgp_inducing* ind,
                   const stgp_neighbors* nb, int policy, stgp_structure** out);
void stgp_structure_destroy(stgp_structure* s);
/* field mirrors for the reference tests (s.D, s.B, s.fitc_diag, s.lambda) */
int stgp_structure_download_D(const stgp_structure* s, double* D_out);
int stgp_structure_download_A(const stgp_structure* s, double* A_out); /* n*m_v, B = I - A on N */
int stgp_structure_download_fitc_diag(const stgp_structure* s, double* diag_out);

/* ---- likelihood, gradient, GLS, prediction (approximations.hpp:102-144) ----
 * y_host == NULL uses the dataset's resident response/covariates.
 * grad order (sigma2, sigma1_2, a, c, alpha, beta, delta) (approximations.hpp:23-25). */
int stgp_nll(stgp_structure* s, const double* y_host, const double* X_host, int p,
             const double* beta, double* out);
int stgp_nll_grad(stgp_structure* s, const double* y_host, const double* X_host, int p,
                  const double* beta, double* grad_out);
/* one build + NLL + gradient, the optimizer's evaluation (estimation.cpp:277-325) */
int stgp_nll_and_grad(stgp_structure* s, const double* y_host, const double* X_host, int p,
                      const double* beta, double* nll_out, double* grad_out);
int stgp_gls_beta(stgp_structure* s, const double* y_host, const double* X_host, int p,
                  double* beta_out);
int stgp_predict(stgp_structure* s, const double* y_host, const double* X_host, int p,
                 const double* beta, int n_p, const double* targets_xyt_host,
                 const double* Xp_host, int pred_m_v, double* mu_out, double* var_out);
/* Rebuild an existing structure at new parameters and evaluate NLL + gradient
 * (reuses all allocations; the hot loop of a fit). */
int stgp_eval(stgp_structure* s, const stgp_params* theta, const double* y_host,
              const double* X_host, int p, const double* beta, double* nll_out,
              double* grad_out);

/* ---- latent-policy likelihoods ----
 * stgp_nll on a latent-policy Vecchia / VIF structure is the Gaussian latent-policy NLL through the
 * Laplace algebra (approximations.cpp:320-334, 348-349, 369-371).  The Laplace algebra factors Q + W
 * densely on the device ("desk scale", n <= 40000; FITC: any n).
 * laplace_marginal (laplace.cpp:115-203, LaplaceAlgebra approximations.cpp:1083-1375) with the
 * zero-censored power-transformed normal likelihood (LikelihoodParams sigma, lambda; y >= 0): the
 * negative Laplace log-marginal, and the state at the mode (mode, grad_at_mode, w: n each, may be NULL).
 * warm (n, may be NULL) is the Newton warm start. */
int stgp_laplace_marginal(stgp_structure* s, const double* y_host, const double* X_host, int p, const double* beta,
                          double lik_sigma, double lik_lambda, const double* warm_host, double* nll_out,
                          double* mode_out, double* grad_at_mode_out, double* w_out, int* iterations_out);

/* zcptn_predict (laplace.cpp:205-259): latent predictive mean / variance at the targets (n_p x 3 host
 * x, y, t) through the LaplaceAlgebra target rows at the Laplace state (grad_at_mode, w from
 * stgp_laplace_marginal), P(Y > 0), and n_samples Monte Carlo draws per target from
 * mt19937_64(mix_seed(seed, p)); samples (may be NULL) is n_p x n_samples column-major. */
int stgp_zcptn_predict(stgp_structure* s, const double* grad_at_mode_host, const double* w_host, int n_p,
                       const double* targets_xyt_host, const double* Xp_host, int p, const double* beta,
                       double lik_sigma, double lik_lambda, int pred_m_v, int n_samples, uint64_t seed,
                       double* mu_latent_out, double* var_latent_out, double* p_rain_out, double* amount_mean_out,
                       double* amount_median_out, double* samples_out);

/* ---- fit driver (estimation.hpp:23-56, estimation.cpp:423-619; Gaussian likelihood) ---- */
/* FitConfig::Method */
#define STGP_FIT_VECCHIA_EUCLID 0
#define STGP_FIT_VECCHIA_CORR 1
#define STGP_FIT_FITC_KMEANSPP 2
#define STGP_FIT_FITC_STS 3
#define STGP_FIT_VIF 4
typedef struct {
  int method, m_v, m, max_iterations;
  double tol_objective, tol_gradient, nu;
  uint64_t seed;
} stgp_fit_config;
/* TraceRow (estimation.hpp:61-66) */
typedef struct {
  int iteration;
  double nll, grad_norm;
  int refresh;
} stgp_trace_row;
/* default_init (estimation.cpp:68-114) on an ordered dataset with host response y (n) and
 * covariates X (n x p column-major). */
int stgp_default_init(const stgp_dataset* ds, const double* y_host, const double* X_host, int p,
                      const stgp_fit_config* config, stgp_params* out);
/* fit (estimation.cpp:423-619), Gaussian path: L-BFGS in the transformed coordinates with selection
 * refresh at power-of-two iterations, NumericError step halving and GLS beta profiling (p > 0).
 * ds is the ordered dataset (FittedModel.data: order it with stgp_order_observations(config.seed)).
 * init may be NULL (default_init).  Up to trace_cap rows of the trace are copied; *n_trace gets
 * the full count. */
int stgp_fit(stgp_dataset* ds, const double* y_host, const double* X_host, int p, const stgp_fit_config* config,
             const stgp_params* init, stgp_params* theta_out, double* beta_out, double* final_nll,
             int* converged, stgp_trace_row* trace_out, int trace_cap, int* n_trace);

/* ---- dataset CSV and neighbour audit formats (dataset.cpp:191-316, neighbors.cpp:336-355) ---- */
typedef struct stgp_table stgp_table; /* a parsed dataset CSV (host memory) */
/* read_dataset_csv: '#' lines skipped, header names x, y, t, value (required), station_id
 * (optional), every other column a covariate; DataError on malformed input. */
int stgp_read_dataset_csv(const char* path, stgp_table** out);
int stgp_table_shape(const stgp_table* tab, int* n, int* p, int* has_stations);
/* columns in file order; X is n x p column-major (any pointer may be NULL) */
int stgp_table_columns(const stgp_table* tab, double* x, double* y, double* t, double* value, double* X);
/* copy station i / covariate name j into buf (NUL-terminated, truncated to cap); returns the full
 * length, -1 when out of range */
int stgp_table_station(const stgp_table* tab, int i, char* buf, int cap);
int stgp_table_covariate_name(const stgp_table* tab, int j, char* buf, int cap);
void stgp_table_destroy(stgp_table* tab);
/* write_dataset_csv (precision 17, "# comment" line when given, covariates named x0..x{p-1}) */
int stgp_write_dataset_csv(const char* path, int n, const double* x, const double* y, const double* t,
                           const double* value, int p, const double* X, const char* const* stations,
                           const char* header_comment);
/* write_neighbor_debug_csv: "i,rank,neighbor_index,distance" rows, each set sorted by
 * (distance, index), with the metric of the search (cli.cpp:516-572) */
int stgp_write_neighbor_debug_csv(const char* path, const stgp_neighbors* nb, const stgp_dataset* ds,
                                  const char* header_comment);

/* ---- diagnostics ---- */
/* device exp port on n inputs (KAT against the host libm) */
int stgp_debug_exp(stgp_ctx* ctx, int n, const double* x_host, double* out);
/* FP64 FMA throughput microbenchmark: returns achieved TFLOP/s (2 flops / DFMA) */
int stgp_debug_fp64_peak(stgp_ctx* ctx, double* tflops);
/* Measured FP64 tensor-core (mma.sync m8n8k4 f64, DMMA) throughput in TFLOP/s. */
int stgp_debug_dmma_peak(stgp_ctx* ctx, double* tflops);
/* Names of the profiled regions recorded so far, newline separated (truncated to cap-1 bytes). */
int stgp_ctx_profile_names(stgp_ctx* ctx, char* buf, int cap);
/* FP64 product C[r][j] = sum_c A[r][c] B[j][c] (row-major host arrays, n x k, m x k -> n x m)
 * through the int8 Ozaki path (emulated = 1) or the DMMA GEMM (emulated = 0); *ms = device time
 * of the product (inputs resident). */
int stgp_debug_gemm_rows(stgp_ctx* ctx, int emulated, long long n, int m, int k, const double* A_host,
                         const double* B_host, double* C_host, double* ms);
/* FP64 product C[j][i] = sum_r A[j + r m] B[i + r m] (column-major m x n host arrays -> m x m,
 * row-major C) through the int8 Ozaki path (emulated = 1) or the DMMA GEMM (emulated = 0). */
int stgp_debug_gemm_cols(stgp_ctx* ctx, int emulated, int m, long long n, const double* A_host,
                         const double* B_host, double* C_host, double* ms);
/* Triangular product C = op(T) B (the W = L_m^-1 U and omega = L_m^-T omega' shape): T m x m lower
 * triangular, B m x n, C m x n, all column-major host arrays; op(T) = T^T when transpose.  mode 0: the
 * DMMA TRMM; 1: the int8 Ozaki rows form with each Y group's K range cut to the triangle; 2: the same
 * over the full K range.  *ms = device time of the product (inputs resident). */
int stgp_debug_trmm(stgp_ctx* ctx, int mode, int transpose, int m, long long n, const double* T_host,
                    const double* B_host, double* C_host, double* ms);
/* device Gneiting covariance / kernel gradient of (h, u) pairs with live factors; grad6_out may be
   NULL (covariances only).  A general nu (outside {0.5, 1.5, 2.5}) evaluates covariances through the
   Bessel-K Matern and returns STGP_ERR_NUMERIC when a gradient is requested (covariance.cpp:79-87). */
int stgp_debug_kernel(stgp_ctx* ctx, const stgp_params* theta, int n, const double* h_host,
                      const double* u_host, double* cov_out, double* grad6_out);

#ifdef __cplusplus
}
#endif
#endif

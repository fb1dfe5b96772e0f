// Built approximation structures (approximations.hpp:33-75) and the helpers
// shared by the Vecchia / FITC / VIF translation units.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "engine.hpp"
#include "rows.cuh"
#include "tiles.cuh"

namespace stgp {

struct Reducer {
  DevBuf<double> part, out;
  void ensure(int blocks, int width);
  std::vector<double> finish(stgp_ctx* ctx, int blocks, int width);
};

// Low-rank state of FITC / VIF structures (all device, column-major).
struct LowRank {
  int M = 0, ldm = 0;            // inducing count, padded leading dimension (multiple of 4)
  std::vector<double> zxyt;      // host M x 3
  DevBuf<double> zx, zy, zt;     // device inducing coordinates
  DevBuf<int32_t> ztid;          // time ids of inducing points
  DevBuf<double> Lm;             // Cholesky of jittered Sigma_m (ldm x ldm, lower)
  double logdet_m = 0.0;
  DevBuf<double> U, W;           // ldm x n : cross covariance, whitened L_m^{-1} U
  DevBuf<double> Vp;             // VIF: V' = W B^T (ldm x n)
  DevBuf<double> Mc;             // Woodbury core (ldm x ldm), Cholesky in place
  double logdet_M = 0.0;
  DevBuf<double> fitc_diag, lambda;  // FITC
  DevBuf<double> Lminv, Kinv;        // explicit inverses of L_m and K (M x M)
  DevBuf<double> Kfull;              // K itself (before its Cholesky), for prediction
  DevBuf<double> Lfac;               // per-row closure Cholesky factors from the build (VIF)
  DevBuf<double> work1, work2, work3, work4, vecM, vecM2, vecN, vecN2;
  std::map<std::string, DevBuf<double>> pool;  // persistent per-structure temporaries
  double* tmp(const char* name, size_t count) {
    DevBuf<double>& b = pool[name];
    b.ensure(count);
    return b.get();
  }
};

}  // namespace stgp

namespace stgp {
struct LaplaceDev;  // laplace.cu: latent-policy Laplace algebra state
}

struct stgp_structure {
  stgp_structure();  // assigns uid
  ~stgp_structure();
  uint64_t uid = 0;  // process-unique, never reused (owner tag of kept Ozaki digits)
  stgp_dataset* ds = nullptr;
  int kind = 0, policy = 0;
  stgp::Params th{};
  int n = 0, m_v = 1;
  int row_begin = 0, row_end = 0;
  int col_begin = 0;  // first column this shard touches (halo of its neighbour sets)
  stgp::DevBuf<int32_t> nbr;
  int nbr_kind = 0;
  double nbr_ss = 1.0, nbr_ts = 1.0;  // Euclidean scales of the neighbour sets (prediction metric)
  stgp::DevBuf<double> A, D;
  stgp::TimeIndex ti;
  bool ti_dirty = true;
  stgp::DevLagTable lt;
  stgp::Reducer red;
  stgp::DevBuf<int> fail;
  stgp::DevBuf<double> r, ywork, Xwork, betaw, u, scratch, row_part;
  stgp::DevBuf<double> pairw;  // two-pass Vecchia gradient: per-row pair weights (rows.cuh kPairW)
  stgp::DevBuf<double> zcol;  // ldw zeros (fragment source of empty closure slots)
  int zcol_n = 0;
  stgp::LowRank lr;
  bool built = false;
  // CSC of B's pattern for deterministic B^T products
  bool csc_built = false;
  stgp::DevBuf<int32_t> csc_ptr, csc_row;
  stgp::DevBuf<int16_t> csc_slot;
  // locality schedule (lowrank.cu: locality_order): rows [row_begin, row_end), columns [col_begin, row_end)
  stgp::DevBuf<int32_t> rorder, corder;
  bool order_rows = false, order_gather = false;
  // tile-staged gathers (tiles.cu), built once per structure
  bool tiles_built = false;
  stgp::TileSets tiles;
  stgp::LaplaceDev* lap = nullptr;  // dense Q + W factor etc. (laplace.cu), per call
};

namespace stgp {

extern thread_local std::string g_last_error;

void compute_residual(stgp_structure* s, const double* y_host, const double* X_host, int p,
                      const double* beta);
RowArgs row_args(stgp_structure* s, const double* W, int ldw, double nugget);
std::vector<double> run_rows(stgp_structure* s, int mode, const double* W, int ldw, double nugget);
std::vector<double> run_rows_args(stgp_structure* s, int mode, RowArgs& a);
void prepare_tables(stgp_structure* s);
double nll_const(int n);
void launch_nll_stored(stgp_structure* s, int blocks, double* u_out);
int row_blocks(stgp_ctx* ctx, int rows);
int lfac_stride_for(int m_v);
unsigned long long* claim_counter(stgp_ctx* ctx);  // zeroed in-order work counter
// exact spatial-tile neighbour search (selection.cu): d_r with inducing points, d_c without
stgp_neighbors* spatial_search(stgp_dataset* ds, const Params& p, const std::vector<double>& zxyt, int m_v, int kind);  // per-row stored closure factor size (doubles)
void upload_lag_table(DevLagTable& d, const TimeIndex& ti, const Params& p, const LagPolicy& pol,
                      cudaStream_t s, bool index_changed);
LagTable lag_view(const DevLagTable& d);
// latent-policy likelihoods (laplace.cu)
void laplace_release(stgp_structure* s);
double latent_policy_nll_dev(stgp_structure* s);
void laplace_prepare_w(stgp_structure* s, const double* w_dev);
void laplace_solve_cols(stgp_structure* s, const double* X, long long ncols, double* out);
void zcptn_moments_dev(stgp_structure* s, const double* a_host, const double* w_host, int np, const double* txyt,
                       int pred_m_v, double* mu_lat, double* var_lat);
double laplace_marginal_dev(stgp_structure* s, const double* y_host, const double* off_dev, double sigma,
                            double lambda, const double* warm_host, double* mode_out, double* a_out, double* w_out,
                            int* iters_out);

}  // namespace stgp

extern "C" void stgp_ctx_release_comm(stgp_ctx* ctx);

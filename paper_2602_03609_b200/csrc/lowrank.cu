// FITC / VIF low-rank algebra (approximations.cpp:217-312, 352-384, 495-744, 923-1080).
#include "comm.hpp"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {
void lowrank_setup(stgp_structure*, const stgp_inducing*) { config_error("FITC/VIF: not built yet"); }
void fitc_build(stgp_structure*) { config_error("FITC: not built yet"); }
void vif_build(stgp_structure*) { config_error("VIF: not built yet"); }
double lowrank_nll(stgp_structure*) { config_error("FITC/VIF: not built yet"); }
void lowrank_nll_grad(stgp_structure*, double*, double*) { config_error("FITC/VIF: not built yet"); }
void lowrank_predict(stgp_structure*, int, const double*, int, double*, double*) { config_error("predict: not built yet"); }
void vecchia_predict(stgp_structure*, int, const double*, int, double*, double*) { config_error("predict: not built yet"); }
std::vector<double> sigma_inv_apply_host(stgp_structure*, const double*) { config_error("gls: not built yet"); }
}  // namespace stgp

extern "C" {
int stgp_residual_neighbors(stgp_dataset*, const stgp_params*, const stgp_inducing*, int, stgp_neighbors**) {
  stgp::g_last_error = "residual_neighbors: not built yet";
  return STGP_ERR_CONFIG;
}
int stgp_inducing_create(stgp_ctx* ctx, int M, const double* xyt, stgp_inducing** out) {
  auto* ind = new stgp_inducing();
  ind->ctx = ctx;
  ind->xyt.assign(xyt, xyt + 3 * static_cast<size_t>(M));
  *out = ind;
  return STGP_OK;
}
int stgp_sts_kmeanspp(stgp_dataset*, int, uint64_t, stgp_inducing**) {
  stgp::g_last_error = "sts_kmeanspp: not built yet";
  return STGP_ERR_CONFIG;
}
int stgp_joint_kmeanspp_inducing(stgp_dataset*, int, double, double, uint64_t, stgp_inducing**) {
  stgp::g_last_error = "joint_kmeanspp: not built yet";
  return STGP_ERR_CONFIG;
}
int stgp_kmeanspp(stgp_ctx*, const double*, int, int, int, uint64_t, double*) {
  stgp::g_last_error = "kmeanspp: not built yet";
  return STGP_ERR_CONFIG;
}
int stgp_inducing_size(const stgp_inducing* ind, int* M, int* m_s, int* m_t) {
  if (M) *M = ind->M();
  if (m_s) *m_s = ind->m_s;
  if (m_t) *m_t = ind->m_t;
  return STGP_OK;
}
int stgp_inducing_download(const stgp_inducing* ind, double* xyt) {
  std::copy(ind->xyt.begin(), ind->xyt.end(), xyt);
  return STGP_OK;
}
void stgp_inducing_destroy(stgp_inducing* ind) { delete ind; }
}

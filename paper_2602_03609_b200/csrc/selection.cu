// Residual-correlation (d_r) neighbour search and space-time kMeans++ seeding.
#include "comm.hpp"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

extern "C" {
int stgp_residual_neighbors(stgp_dataset*, const stgp_params*, const stgp_inducing*, int, stgp_neighbors**) {
  stgp::g_last_error = "residual_neighbors: not built yet";
  return STGP_ERR_CONFIG;
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
}

// Prediction and GLS (approximations.cpp:752-1080).
#include "comm.hpp"
#include "dense.cuh"
#include "lowrank_common.cuh"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {
void lowrank_predict(stgp_structure*, int, const double*, int, double*, double*) { config_error("predict: not built yet"); }
void vecchia_predict(stgp_structure*, int, const double*, int, double*, double*) { config_error("predict: not built yet"); }
std::vector<double> sigma_inv_apply_host(stgp_structure*, const double*) { config_error("gls: not built yet"); }
}  // namespace stgp

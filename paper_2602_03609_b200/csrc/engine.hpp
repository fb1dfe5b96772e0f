// Host-side engine objects behind the C ABI (include/stgp_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "gneiting.cuh"

struct ncclComm;

namespace stgp {

// ---- host replicas of the reference's scalar functions (glibc, no FMA) ----
void validate_params(const Params& p);              // covariance.cpp:34-46
TF host_factors(const Params& p, double u);          // covariance.cpp:94-113
void host_grad00(const Params& p, double g[6]);      // GneitingKernel::grad(0, 0)
void require_analytic_grad(const Params& p);        // NumericError for general nu (covariance.cpp:79-87)
DevKernel dev_kernel(const Params& p);
constexpr int kMaxSearchM = 128;  // neighbour lists of up to 4 slots per lane (search.cuh topl_*)
uint64_t mix_seed(uint64_t seed, uint64_t stream);   // types.hpp:65-70

// Distinct-time groups of one computation (data times, then inducing times,
// then prediction targets).  lagid maps every time-id pair to a distinct lag
// value; temporal factors are tabulated per distinct lag.
struct TimeIndex {
  std::vector<double> T;      // concatenated group times
  std::vector<double> lags;   // distinct |T_a - T_b|
  std::vector<int32_t> lagid; // nT * nT
  int nT() const { return static_cast<int>(T.size()); }
  void build();
};

// The integer-lag table of a structure kernel (approximations.cpp:26-38):
// present when every data time is integral to 1e-9 and the range <= 2e5.
struct LagPolicy {
  bool table = false;
  int size = 0;  // entries 0..size-1
};
std::vector<TF> tabulate(const Params& p, const std::vector<double>& lags, const LagPolicy& pol);

struct DevLagTable {
  DevBuf<int32_t> lagid;
  DevBuf<TF> tf;
  int nT = 0;
  std::vector<TF> host_tf;
  // live mode (more than kMaxTableTimes distinct times): time values, integer-lag table, parameters
  bool live = false;
  DevBuf<double> Tv;
  DevBuf<TF> itab;
  int itab_n = 0;
  double la = 0.0, two_alpha = 0.0, E = 0.0, half_beta = 0.0;
};
constexpr int kMaxTableTimes = 4096;  // nT x nT lag ids above this: live factors

struct OzakiState;  // ozaki.cu: int8 slice buffers and the tcgen05 kernel work lists
}  // namespace stgp

struct stgp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  ncclComm* comm = nullptr;
  int64_t launches = 0;
  int num_sms = 148;
  int (*host_allreduce)(void*, double*, int64_t) = nullptr;  // stgp_ctx_set_host_allreduce
  void* host_allreduce_user = nullptr;
  stgp::DevBuf<int> iscr;     // small persistent scratch (flags, scalars)
  stgp::DevBuf<double> dscr;
  stgp::DevBuf<double> gemm_part;  // split-K partial tiles of the DMMA GEMM
  stgp::DevBuf<double> dense_tmp;  // GEMV partials, transposed TRSM operands, Cholesky panels
  stgp::DevBuf<double> dense_tmp2;  // blocked TRSM: one row block of the solution
  stgp::DevBuf<double> dense_inv;   // inverses of the 64 x 64 diagonal blocks of a factor
  stgp::DevBuf<double> dense_tmp3;  // n x n: triangular inverse / congruence product
  stgp::DevBuf<double> sel_W;  // d_r search: whitened cross covariance, kept across searches (8 GB at cfg4)
  stgp::DevBuf<uint16_t> sel_W16;  // d_r search: its fp16 copy for the certified filter
  stgp::OzakiState* ozaki = nullptr;  // FP64-on-int8 GEMM workspace (lazy)
  // live per-region kernel timing (stgp_ctx_profile)
  bool prof = false;
  std::map<std::string, std::pair<double, int64_t>> prof_acc;
  std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> prof_pending;
  std::vector<cudaEvent_t> prof_events;  // collected events, reused (no driver calls per region)
};

namespace stgp {
// Records an event pair around the launches issued in its scope (when profiling).
struct ProfRegion {
  stgp_ctx* ctx;
  const char* name;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ProfRegion(stgp_ctx* c, const char* n);
  ~ProfRegion();
};
// Collect pending event pairs after a stream synchronisation.
void prof_collect(stgp_ctx* ctx);
}  // namespace stgp

struct stgp_dataset {
  stgp_ctx* ctx = nullptr;
  int n = 0;
  std::vector<double> hx, hy, ht;
  stgp::DevBuf<double> x, y, t;
  stgp::DevBuf<int32_t> tid;  // index into Tdata
  std::vector<double> Tdata;  // distinct data times ascending
  std::vector<int32_t> htid;
  bool time_sorted = false;
  stgp::DevBuf<int32_t> blk_start;  // (time sorted) start of each equal-time block, size nT+1
  stgp::LagPolicy lagpol;
  // resident response / covariates
  stgp::DevBuf<double> resp, X;
  int p = 0;
  bool has_resp = false;
  // spatial-tile search meta (selection.cu), computed on first use under tile_mu: time buckets and
  // bounding box
  std::mutex tile_mu;
  bool tile_meta = false;
  std::vector<int> tile_bstart;
  double tile_x0 = 0, tile_x1 = 0, tile_y0 = 0, tile_y1 = 0;
};

struct stgp_neighbors {
  stgp_ctx* ctx = nullptr;
  int n = 0, m_v = 0, kind = 0;
  stgp::DevBuf<int32_t> idx;
  stgp::DevBuf<double> dist;
  bool has_dist = false;
  double ss = 1.0, ts = 1.0;
};

struct stgp_inducing {
  stgp_ctx* ctx = nullptr;
  std::vector<double> xyt;  // M x 3 row-major
  int m_s = 0, m_t = 0;
  int M() const { return static_cast<int>(xyt.size() / 3); }
};

struct stgp_structure;

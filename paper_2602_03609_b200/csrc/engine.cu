// Host orchestration of the stgp B200 engine and the C ABI (include/stgp_b200.h).
//
// Host code here only sequences device work, tabulates per-lag temporal factors
// with glibc (bit-identical to the reference's pow/log) and moves O(1)-sized
// results.  Every O(n) loop of the hot path runs in a CUDA kernel.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <numeric>
#include <random>
#include <set>

#include "comm.hpp"
#include "dense.cuh"
#include "engine.hpp"
#include "ozaki.cuh"
#include "rows.cuh"
#include "rows_serial.cuh"
#include "search.cuh"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

namespace {
struct PoolDev {
  bool init = false;
  bool on = false;
  cudaMemPool_t pool = nullptr;
  cudaStream_t stream = nullptr;  // private, idle between calls: allocations are ready on return
};
PoolDev g_pool[64];
std::mutex g_pool_mu;

PoolDev& pool_dev(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  PoolDev& d = g_pool[dev & 63];
  if (!d.init) {
    d.init = true;
    const char* e = std::getenv("STGP_POOL");
    d.on = !(e && e[0] == '0');
    if (d.on) {
      // The device's default pool with an unbounded release threshold.  A private pool (cudaMemPoolCreate)
      // was tried: its first growth made the cold cfg4 d_r search 1.75 s instead of 0.49 s
      // (scripts/search_cold_probe.py), so the default pool stays; STGP_POOL=0 restores cudaMalloc.
      STGP_CUDA(cudaDeviceGetDefaultMemPool(&d.pool, dev));
      uint64_t thr = UINT64_MAX;
      STGP_CUDA(cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &thr));
      STGP_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    }
  }
  return d;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  int dev = 0;
  STGP_CUDA(cudaGetDevice(&dev));
  PoolDev& d = pool_dev(dev);
  void* p = nullptr;
  if (!d.on) {
    STGP_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  cudaError_t e = cudaMallocFromPoolAsync(&p, bytes, d.pool, d.stream);
  if (e == cudaErrorMemoryAllocation) {  // cached blocks of other sizes: hand them back and retry
    (void)cudaGetLastError();
    STGP_CUDA(cudaDeviceSynchronize());
    STGP_CUDA(cudaMemPoolTrimTo(d.pool, 0));
    e = cudaMallocFromPoolAsync(&p, bytes, d.pool, d.stream);
  }
  STGP_CUDA(e);
  STGP_CUDA(cudaStreamSynchronize(d.stream));
  return p;
}

void dev_free(void* p) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  PoolDev& d = pool_dev(dev);
  if (!d.on) {
    cudaFree(p);
    return;
  }
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) == cudaSuccess && a.device != dev) {
    cudaSetDevice(a.device);
    dev_free(p);
    cudaSetDevice(dev);
    return;
  }
  cudaDeviceSynchronize();  // cudaFree semantics: no stream may still be using the block
  cudaFreeAsync(p, d.stream);
}


thread_local std::string g_last_error;

void validate_params(const Params& p) {
  auto fail = [](const char* w) { config_error(std::string("CovarianceParams: ") + w); };
  if (!(p.sigma2 >= 0.0) || !std::isfinite(p.sigma2)) fail("sigma2 must be >= 0");
  if (!(p.sigma1_2 > 0.0) || !std::isfinite(p.sigma1_2)) fail("sigma1_2 must be > 0");
  if (!(p.a > 0.0) || !std::isfinite(p.a)) fail("a must be > 0");
  if (!(p.c > 0.0) || !std::isfinite(p.c)) fail("c must be > 0");
  if (!(p.alpha > 0.0 && p.alpha <= 1.0)) fail("alpha must be in (0, 1]");
  if (!(p.nu > 0.0) || !std::isfinite(p.nu)) fail("nu must be > 0");
  if (!(p.beta >= 0.0 && p.beta <= 1.0)) fail("beta must be in [0, 1]");
  if (!(p.delta >= 0.0) || !std::isfinite(p.delta)) fail("delta must be >= 0");
}

static double exponent_E(const Params& p) { return p.delta + p.beta * 2 / 2.0; }

TF host_factors(const Params& p, double u) {
  TF f;
  if (u == 0.0) {
    f.u2a = 0.0;
    f.u2a_logu = 0.0;
    f.pow_mE = 1.0;
    f.pow_mbh = 1.0;
    f.inv_T = 1.0;
    f.log_T = 0.0;
    return f;
  }
  f.u2a = std::pow(u, 2.0 * p.alpha);
  f.u2a_logu = f.u2a * std::log(u);
  const double T = p.a * f.u2a + 1.0;
  f.inv_T = 1.0 / T;
  f.log_T = std::log(T);
  f.pow_mE = std::pow(T, -exponent_E(p));
  f.pow_mbh = std::pow(T, -p.beta / 2.0);
  return f;
}

// GneitingKernel::grad -> matern_corr_deriv (covariance.cpp:79-87): analytic only for the closed forms
void require_analytic_grad(const Params& p) {
  if (nu_code_of(p.nu) == kNuGeneral)
    numeric_error(
        "matern_corr_deriv: analytic derivative only for nu in {0.5, 1.5, 2.5}; use finite differences for "
        "general nu");
}

void host_grad00(const Params& p, double g[6]) {
  // GneitingKernel::grad(0, 0): x = 0, M = 1, M' = matern_corr_deriv(0)
  const double x = 0.0;
  const double M = 1.0;
  const double Mp = p.nu == 0.5 ? -1.0 : (p.nu == 1.5 ? -x * 1.0 : -(x * (1.0 + x) / 3.0) * 1.0);
  const double base = p.sigma1_2 * 1.0;
  const double E = exponent_E(p);
  g[0] = 1.0 * M;
  const double dC_dT = base * 1.0 * (-E * M - 0.5 * p.beta * x * Mp);
  g[1] = dC_dT * 0.0;
  g[3] = dC_dT * 2.0 * p.a * 0.0;
  g[2] = base * Mp * x / p.c;
  g[4] = -0.0 * base * (M + 0.5 * x * Mp);
  g[5] = -0.0 * base * M;
}

DevKernel dev_kernel(const Params& p) {
  DevKernel k;
  k.s1 = p.sigma1_2;
  k.c = p.c;
  k.a = p.a;
  k.beta = p.beta;
  k.E = exponent_E(p);
  k.nu_code = nu_code_of(p.nu);
  k.g = MaternNu{};
  if (k.nu_code == kNuGeneral) {
    // constants of the general Matern (covariance.cpp:73-74) and Temme's Gamma combinations at mu
    MaternNu& g = k.g;
    g.nu = p.nu;
    g.coef = std::pow(2.0, 1.0 - p.nu) / std::tgamma(p.nu);
    g.nl = static_cast<int>(p.nu + 0.5);
    g.mu = p.nu - g.nl;
    constexpr double kEps = 2.220446049250313e-16;
    g.gampl = 1.0 / std::tgamma(1.0 + g.mu);
    g.gammi = 1.0 / std::tgamma(1.0 - g.mu);
    g.gam1 = std::fabs(g.mu) < kEps ? -0.5772156649015328606 : (g.gammi - g.gampl) / (2.0 * g.mu);
    g.gam2 = (g.gammi + g.gampl) / 2.0;
    const double pimu = 3.141592653589793 * g.mu;
    g.fact = std::fabs(pimu) < kEps ? 1.0 : pimu / std::sin(pimu);
  }
  return k;
}

uint64_t mix_seed(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void TimeIndex::build() {
  const int nt = nT();
  if (nt > kMaxTableTimes) {  // live mode: the device evaluates each pair's lag (upload_lag_table)
    lags.clear();
    lagid.clear();
    return;
  }
  std::vector<double> all;
  all.reserve(static_cast<size_t>(nt) * (nt + 1) / 2);
  for (int a = 0; a < nt; ++a)
    for (int b = 0; b <= a; ++b) all.push_back(std::abs(T[static_cast<size_t>(a)] - T[static_cast<size_t>(b)]));
  std::sort(all.begin(), all.end());
  all.erase(std::unique(all.begin(), all.end()), all.end());
  lags = all;
  lagid.assign(static_cast<size_t>(nt) * nt, 0);
  for (int a = 0; a < nt; ++a)
    for (int b = 0; b <= a; ++b) {
      const double u = std::abs(T[static_cast<size_t>(a)] - T[static_cast<size_t>(b)]);
      const int id = static_cast<int>(std::lower_bound(lags.begin(), lags.end(), u) - lags.begin());
      lagid[static_cast<size_t>(a) * nt + b] = id;
      lagid[static_cast<size_t>(b) * nt + a] = id;
    }
}

std::vector<TF> tabulate(const Params& p, const std::vector<double>& lags, const LagPolicy& pol) {
  std::vector<TF> out(lags.size());
  for (size_t i = 0; i < lags.size(); ++i) {
    const double u = lags[i];
    if (pol.table) {  // covariance.cpp:127-146 snap rule
      const double r = std::nearbyint(u);
      if (std::abs(u - r) < 1e-9 && r >= 0.0 && static_cast<int>(r) < pol.size) {
        out[i] = host_factors(p, static_cast<double>(static_cast<int>(r)));
        continue;
      }
    }
    out[i] = host_factors(p, u);
  }
  return out;
}

void upload_lag_table(DevLagTable& d, const TimeIndex& ti, const Params& p, const LagPolicy& pol,
                      cudaStream_t s, bool index_changed) {
  if (ti.nT() > kMaxTableTimes) {
    d.live = true;
    if (index_changed || d.nT != ti.nT()) {
      d.Tv.upload(ti.T.data(), ti.T.size(), s);
      d.nT = ti.nT();
    }
    // the integer-lag table of the policy (host glibc), bit-identical to the table mode
    d.itab_n = pol.table ? pol.size : 0;
    if (d.itab_n > 0) {
      std::vector<double> ul(static_cast<size_t>(d.itab_n));
      for (int u = 0; u < d.itab_n; ++u) ul[static_cast<size_t>(u)] = u;
      LagPolicy none;
      d.host_tf = tabulate(p, ul, none);
      d.itab.upload(d.host_tf.data(), d.host_tf.size(), s);
    }
    d.la = p.a;
    d.two_alpha = 2.0 * p.alpha;
    d.E = exponent_E(p);
    d.half_beta = p.beta / 2.0;
    return;
  }
  d.live = false;
  if (index_changed || d.nT != ti.nT()) {
    d.lagid.upload(ti.lagid.data(), ti.lagid.size(), s);
    d.nT = ti.nT();
  }
  d.host_tf = tabulate(p, ti.lags, pol);
  d.tf.upload(d.host_tf.data(), d.host_tf.size(), s);
}

LagTable lag_view(const DevLagTable& d) {
  if (d.live)
    return LagTable{nullptr, nullptr, d.nT, d.Tv.get(), d.itab_n > 0 ? d.itab.get() : nullptr, d.itab_n,
                    d.la, d.two_alpha, d.E, d.half_beta};
  return LagTable{d.lagid.get(), d.tf.get(), d.nT, nullptr, nullptr, 0, 0.0, 0.0, 0.0, 0.0};
}

ProfRegion::ProfRegion(stgp_ctx* c, const char* n) : ctx(c), name(n) {
  if (!ctx->prof) return;
  for (cudaEvent_t* e : {&e0, &e1}) {
    if (!ctx->prof_events.empty()) {
      *e = ctx->prof_events.back();
      ctx->prof_events.pop_back();
    } else {
      cudaEventCreate(e);
    }
  }
  cudaEventRecord(e0, ctx->stream);
}
ProfRegion::~ProfRegion() {
  if (!e0) return;
  cudaEventRecord(e1, ctx->stream);
  ctx->prof_pending.push_back({name, {e0, e1}});
}
void prof_collect(stgp_ctx* ctx) {
  for (auto& p : ctx->prof_pending) {
    cudaEventSynchronize(p.second.second);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.second.first, p.second.second);
    auto& acc = ctx->prof_acc[p.first];
    acc.first += ms;
    acc.second += 1;
    ctx->prof_events.push_back(p.second.first);
    ctx->prof_events.push_back(p.second.second);
  }
  ctx->prof_pending.clear();
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
__global__ void residual_kernel(int n, const double* y, const double* X, int p, const double* beta, double* r) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double xb = 0.0;
    for (int j = 0; j < p; ++j) xb += X[static_cast<size_t>(i) + static_cast<size_t>(j) * n] * beta[j];
    r[i] = y[i] - xb;
  }
}

// u_i = (B r)_i from stored A; NLL terms log D + u^2 / D (approximations.cpp:336-347)
__global__ void __launch_bounds__(256) vecchia_nll_stored_kernel(int row_begin, int row_end, int m_v,
                                                                  const int32_t* nbr, const double* A,
                                                                  const double* D, const double* r,
                                                                  double* u_out, double* part) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int i = row_begin + blockIdx.x * blockDim.x + threadIdx.x; i < row_end; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int a = 0; a < m_v; ++a) {
      const int j = nbr[static_cast<size_t>(i) * m_v + a];
      if (j < 0) break;
      s += -A[static_cast<size_t>(i) * m_v + a] * r[j];
    }
    const double u = s + r[i];
    if (u_out) u_out[i] = u;
    acc += log(D[i]) + u * u / D[i];
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// 16 independent DFMA chains per thread
__global__ void fp64_peak_kernel(int iters, double* out) {
  double a[16];
  const double m = 1.0000001, c = 1e-9;
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = threadIdx.x * 1e-3 + q;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 16; ++q) a[q] = fma(a[q], m, c);
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 16; ++q) s += a[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 8 independent m8n8k4 f64 MMA chains per warp (512 flop each)
__global__ void dmma_peak_kernel(int iters, double* out) {
  double d[8][2];
  const double a = 1.0 + threadIdx.x * 1e-7, b = 0.999999;
#pragma unroll
  for (int q = 0; q < 8; ++q) d[q][0] = d[q][1] = q * 1e-3;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[q][0]), "+d"(d[q][1])
                   : "d"(a), "d"(b));
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += d[q][0] + d[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void debug_exp_kernel(int n, const double* x, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = glibc_exp(x[i]);
}

__global__ void debug_kernel_kernel(int n, DevKernel k, const TF* tf, const double* h, double* cov, double* g6) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double g[6];
    const TF f = tf[i];
    cov[i] = gneiting_eval<true>(k, h[i], f);
    if (!g6) continue;
    gneiting_grad(k, h[i], f, g);
    for (int q = 0; q < 6; ++q) g6[static_cast<size_t>(i) * 6 + q] = g[q];
  }
}

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
void Reducer::ensure(int blocks, int width) {
  part.ensure(static_cast<size_t>(blocks) * width);
  out.ensure(static_cast<size_t>(width));
}
std::vector<double> Reducer::finish(stgp_ctx* ctx, int blocks, int width) {
  if (width < 1 || width > 8) throw Error(kInternal, "Reducer: width must lie in [1, 8]");
  reduce_parts_kernel<<<1, 32 * width, 0, ctx->stream>>>(part.get(), blocks, width, out.get());
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
  std::vector<double> h(static_cast<size_t>(width));
  out.download(h.data(), h.size(), ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

int lfac_stride_for(int m_v) {
  const int ks = m_v <= 8 ? 8 : (m_v <= 16 ? 16 : (m_v <= 24 ? 24 : 31));
  return ks * (ks + 1) / 2 + 32;
}

int row_blocks(stgp_ctx* ctx, int rows) {
  const int need = ceil_div(std::max(rows, 1), kRowWarps);
  return std::max(1, std::min(need, ctx->num_sms * 16));
}

}  // namespace stgp

using namespace stgp;

// ===========================================================================
// structure internals shared with the other translation units
// ===========================================================================
namespace stgp {

void compute_residual(stgp_structure* s, const double* y_host, const double* X_host, int p,
                      const double* beta) {
  stgp_ctx* ctx = s->ds->ctx;
  const int n = s->n;
  s->r.ensure(static_cast<size_t>(n));
  const double* yd;
  const double* Xd = nullptr;
  int pp = 0;
  if (y_host) {
    s->ywork.upload(y_host, static_cast<size_t>(n), ctx->stream);
    yd = s->ywork.get();
    if (p > 0 && beta) {
      s->Xwork.upload(X_host, static_cast<size_t>(n) * p, ctx->stream);
      Xd = s->Xwork.get();
      pp = p;
    }
  } else {
    if (!s->ds->has_resp) config_error("no response: pass y or call stgp_dataset_set_response");
    yd = s->ds->resp.get();
    if (p > 0 && beta) {
      if (p != s->ds->p) config_error("beta length does not match X");
      Xd = s->ds->X.get();
      pp = p;
    }
  }
  if (pp > 0) s->betaw.upload(beta, static_cast<size_t>(pp), ctx->stream);
  residual_kernel<<<std::min(ceil_div(n, 256), 1024), 256, 0, ctx->stream>>>(n, yd, Xd, pp, s->betaw.get(), s->r.get());
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
}

RowArgs row_args(stgp_structure* s, const double* W, int ldw, double nugget) {
  RowArgs a{};
  a.n = s->n;
  a.m_v = s->m_v;
  a.row_begin = s->row_begin;
  a.row_end = s->row_end;
  a.order = s->order_rows ? s->rorder.get() : nullptr;
  a.nbr = s->nbr.get();
  a.x = s->ds->x.get();
  a.y = s->ds->y.get();
  a.tid = s->ds->tid.get();
  a.k = dev_kernel(s->th);
  a.lt = lag_view(s->lt);
  a.s1 = s->th.sigma1_2;
  a.nugget = nugget;
  a.W = W;
  a.ldw = ldw;
  if (W) {
    if (s->zcol_n < ldw) {
      s->zcol.alloc(static_cast<size_t>(ldw));
      s->zcol.zero(s->ds->ctx->stream);
      s->zcol_n = ldw;
    }
    a.zcol = s->zcol.get();
  }
  a.r = s->r.get();
  a.A_out = s->A.get();
  a.D_out = s->D.get();
  a.fail_row = s->fail.get();
  a.u_out = nullptr;
  a.Lfac_out = nullptr;
  a.Lfac_in = nullptr;
  a.A_in = nullptr;
  a.Ga_in = nullptr;
  a.inv_c = 1.0 / s->th.c;
  host_grad00(s->th, a.g00);
  return a;
}

// zeroed work counter for kernels that claim their items in order
unsigned long long* claim_counter(stgp_ctx* ctx) {
  DevBuf<int>& ctr = ctx->iscr;
  ctr.ensure(2);
  STGP_CUDA(cudaMemsetAsync(ctr.get(), 0, sizeof(unsigned long long), ctx->stream));
  return reinterpret_cast<unsigned long long*>(ctr.get());
}

// Launch a warp-per-row kernel: the static grid, or (a.next set) one resident wave whose warps
// claim rows in schedule order.
template <typename K>
static int launch_row_kernel(stgp_ctx* ctx, K kern, int static_blocks, RowArgs& a) {
  int blocks = static_blocks;
  if (a.next) {
    int per_sm = 0;
    STGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowWarps * 32, 0));
    blocks = std::max(1, std::min(per_sm, 16)) * ctx->num_sms;
  }
  kern<<<blocks, kRowWarps * 32, 0, ctx->stream>>>(a);
  return blocks;
}

// Vecchia gradient in two kernels (factor pass, pair pass); STGP_VGRAD_SPLIT=0 runs the fused kernel
static bool vgrad_split() {
  static const bool on = [] {
    const char* e = std::getenv("STGP_VGRAD_SPLIT");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// Launch the per-row kernel in the given mode; returns the 8 reduced partials.
std::vector<double> run_rows(stgp_structure* s, int mode, const double* W, int ldw, double nugget) {
  RowArgs a = row_args(s, W, ldw, nugget);
  return run_rows_args(s, mode, a);
}

std::vector<double> run_rows_args(stgp_structure* s, int mode, RowArgs& a) {
  stgp_ctx* ctx = s->ds->ctx;
  const int rows = s->row_end - s->row_begin;
  int fail_init = INT_MAX;
  s->fail.upload(&fail_init, 1, ctx->stream);
  const bool hw = a.W != nullptr;
  int blocks;
  {
    ProfRegion pr(ctx, mode == kModeVifGrad ? "rows_vifgrad" : "rows");
    if (s->m_v <= kKmax - 1) {
      blocks = row_blocks(ctx, rows);
      s->red.ensure(ctx->num_sms * 16, 8);
      a.part = s->red.part.get();
      // low-rank row kernels gather W columns: ordered claiming keeps them L2-resident
      if (hw && (mode == kModeBuild || mode == kModeVifGrad) && rows > 0) {
        a.next = claim_counter(ctx);
        if (mode != kModeBuild) {
          s->row_part.ensure(static_cast<size_t>(rows) * 8);
          STGP_CUDA(cudaMemsetAsync(s->row_part.get(), 0, sizeof(double) * rows * 8, ctx->stream));
          a.row_part = s->row_part.get();
        }
      }
      const int ks = s->m_v <= 8 ? 8 : (s->m_v <= 16 ? 16 : (s->m_v <= 24 ? 24 : 31));
#define STGP_ROWS(M, HW, KS, ...) blocks = launch_row_kernel(ctx, vecchia_rows_kernel<M, HW, KS, ##__VA_ARGS__>, blocks, a)
#define STGP_ROWS_KS(M, HW)              \
  switch (ks) {                          \
    case 8: STGP_ROWS(M, HW, 8); break;   \
    case 16: STGP_ROWS(M, HW, 16); break; \
    case 24: STGP_ROWS(M, HW, 24); break; \
    default: STGP_ROWS(M, HW, 31); break; \
  }
      if (a.k.nu_code == kNuGeneral) {  // value modes only: the gradient needs a closed-form Matern
        if (mode != kModeBuild && mode != kModeNll) require_analytic_grad(s->th);
        if (mode == kModeBuild) { if (hw) STGP_ROWS(kModeBuild, true, 31, true); else STGP_ROWS(kModeBuild, false, 31, true); }
        else { if (hw) STGP_ROWS(kModeNll, true, 31, true); else STGP_ROWS(kModeNll, false, 31, true); }
      } else if (mode == kModeVifGrad && a.Lfac_in) {
        switch (ks) {
          case 8: blocks = launch_row_kernel(ctx, vif_grad_stored_kernel<8>, blocks, a); break;
          case 16: blocks = launch_row_kernel(ctx, vif_grad_stored_kernel<16>, blocks, a); break;
          case 24: blocks = launch_row_kernel(ctx, vif_grad_stored_kernel<24>, blocks, a); break;
          default: blocks = launch_row_kernel(ctx, vif_grad_stored_kernel<31>, blocks, a); break;
        }
      } else if (mode == kModeBuild) { if (hw) { STGP_ROWS_KS(kModeBuild, true) } else { STGP_ROWS_KS(kModeBuild, false) } }
      else if (mode == kModeNll) { if (hw) { STGP_ROWS_KS(kModeNll, true) } else { STGP_ROWS_KS(kModeNll, false) } }
      else if (mode == kModeGrad && !hw && vgrad_split()) {
        // two passes: factors + pair weights (registers of the Cholesky), then the pair loop at higher
        // occupancy; the second kernel's block partials follow the first's in the reducer
        s->pairw.ensure(static_cast<size_t>(s->n) * kPairW);
        a.pairw = s->pairw.get();
        s->red.ensure(2 * ctx->num_sms * 16, 8);  // both passes' partials (no reallocation in between)
        a.part = s->red.part.get();
        STGP_ROWS_KS(kModeGrad, false)
        RowArgs a2 = a;
        auto pass2 = [&](auto kern) {
          int per_sm = 0;
          STGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowWarps * 32, 0));
          const int b2 = std::max(1, std::min({ceil_div(std::max(rows, 1), kRowWarps), std::max(per_sm, 1) * ctx->num_sms,
                                               ctx->num_sms * 16}));
          a2.part = s->red.part.get() + static_cast<size_t>(blocks) * 8;
          kern<<<b2, kRowWarps * 32, 0, ctx->stream>>>(a2);
          ++ctx->launches;
          blocks += b2;
        };
        switch (ks) {
          case 8: pass2(vecchia_pair_grad_kernel<8>); break;
          case 16: pass2(vecchia_pair_grad_kernel<16>); break;
          case 24: pass2(vecchia_pair_grad_kernel<24>); break;
          default: pass2(vecchia_pair_grad_kernel<31>); break;
        }
      }
      else if (mode == kModeGrad) { if (hw) { STGP_ROWS_KS(kModeGrad, true) } else { STGP_ROWS_KS(kModeGrad, false) } }
      else { STGP_ROWS_KS(kModeVifGrad, true) }
#undef STGP_ROWS_KS
#undef STGP_ROWS
    } else {
      const int threads = 64;
      blocks = std::max(1, std::min(ceil_div(rows, threads), 64));
      const size_t K = static_cast<size_t>(s->m_v);
      const size_t slab = K * K + 8 * K + 16;
      s->scratch.ensure(slab * threads * blocks);
      s->red.ensure(blocks, 8);
      a.part = s->red.part.get();
#define STGP_ROWS(M, HW) vecchia_rows_serial_kernel<M, HW><<<blocks, threads, 0, ctx->stream>>>(a, s->scratch.get())
      if (mode == kModeBuild) { if (hw) STGP_ROWS(kModeBuild, true); else STGP_ROWS(kModeBuild, false); }
      else if (mode == kModeNll) { if (hw) STGP_ROWS(kModeNll, true); else STGP_ROWS(kModeNll, false); }
      else if (mode == kModeGrad) { if (hw) STGP_ROWS(kModeGrad, true); else STGP_ROWS(kModeGrad, false); }
      else STGP_ROWS(kModeVifGrad, true);
#undef STGP_ROWS
    }
  }
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
  if (a.row_part) {  // fixed-order reduction of the per-row contributions
    const int rb2 = std::max(1, std::min(ceil_div(rows, 1024), 1024));
    const int chunk = ceil_div(rows, rb2);
    row_part_reduce_kernel<<<rb2, 256, 0, ctx->stream>>>(a.row_part, rows, chunk, s->red.part.get());
    ++ctx->launches;
    STGP_LAUNCH_CHECK();
    blocks = rb2;
  }
  std::vector<double> tot = s->red.finish(ctx, blocks, 8);
  prof_collect(ctx);
  int fail = 0;
  s->fail.download(&fail, 1, ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  // Agree on failure across shards before anyone raises: a rank that throws alone would leave the
  // others blocked in the next collective, and the fit's line search (estimation.cpp:575-579) needs
  // the NumericError on every rank to halve the step in lockstep.
  std::vector<double> flag{fail != INT_MAX ? 1.0 : 0.0};
  allreduce_host(ctx, flag);
  if (flag[0] > 0.0) {
    if (fail != INT_MAX)
      numeric_error("vecchia row " + std::to_string(fail) +
                    ": conditioning block is not positive definite or non-positive conditional variance");
    numeric_error("vecchia rows of another shard: conditioning block is not positive definite or non-positive "
                  "conditional variance");
  }
  return tot;
}

void prepare_tables(stgp_structure* s) {
  // structure kernel: integer-lag table per maybe_precompute_lags
  upload_lag_table(s->lt, s->ti, s->th, s->ds->lagpol, s->ds->ctx->stream, s->ti_dirty);
  s->ti_dirty = false;
}

double nll_const(int n) { return n * 1.8378770664093453; }

void launch_nll_stored(stgp_structure* s, int blocks, double* u_out) {
  stgp_ctx* ctx = s->ds->ctx;
  vecchia_nll_stored_kernel<<<blocks, 256, 0, ctx->stream>>>(s->row_begin, s->row_end, s->m_v, s->nbr.get(), s->A.get(),
                                                             s->D.get(), s->r.get(), u_out, s->red.part.get());
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
}

}  // namespace stgp

// ===========================================================================
// C ABI
// ===========================================================================
namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return STGP_OK;
  } catch (const stgp::Error& e) {
    stgp::g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    stgp::g_last_error = "out of host memory";
    return STGP_ERR_INTERNAL;
  } catch (const std::exception& e) {
    stgp::g_last_error = e.what();
    return STGP_ERR_INTERNAL;
  }
}

void require(bool c, const char* m) {
  if (!c) config_error(m);
}

}  // namespace

extern "C" {

const char* stgp_last_error(void) { return stgp::g_last_error.c_str(); }
int stgp_version(void) { return 1; }

int stgp_ctx_create(int device, stgp_ctx** out) {
  return guarded([&] {
    require(out != nullptr, "stgp_ctx_create: null out");
    int count = 0;
    STGP_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) config_error("stgp_ctx_create: no such CUDA device");
    STGP_CUDA(cudaSetDevice(device));
    auto ctx = std::make_unique<stgp_ctx>();
    ctx->device = device;
    STGP_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    cudaDeviceProp prop{};
    STGP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      config_error("stgp_b200 is built for sm_100a (B200); found compute capability " +
                   std::to_string(prop.major) + "." + std::to_string(prop.minor));
    ctx->num_sms = prop.multiProcessorCount;
    *out = ctx.release();
  });
}

void stgp_ctx_destroy(stgp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  stgp_ctx_release_comm(ctx);
  stgp::ozaki_release(ctx);
  stgp::prof_collect(ctx);
  for (cudaEvent_t e : ctx->prof_events) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int stgp_ctx_synchronize(stgp_ctx* ctx) {
  return guarded([&] { STGP_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int stgp_ctx_set_shard(stgp_ctx* ctx, int rank, int world) {
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world) config_error("stgp_ctx_set_shard: bad rank/world");
    ctx->rank = rank;
    ctx->world = world;
  });
}

int64_t stgp_ctx_kernel_launches(const stgp_ctx* ctx) { return ctx ? ctx->launches : 0; }
void* stgp_ctx_stream(stgp_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int stgp_ctx_profile(stgp_ctx* ctx, int enable) {
  return guarded([&] {
    require(ctx, "null context");
    ctx->prof = enable != 0;
  });
}
int stgp_ctx_profile_get(stgp_ctx* ctx, const char* region, double* total_ms, int64_t* count) {
  return guarded([&] {
    require(ctx && region, "null argument");
    prof_collect(ctx);
    auto it = ctx->prof_acc.find(region);
    *total_ms = it == ctx->prof_acc.end() ? 0.0 : it->second.first;
    *count = it == ctx->prof_acc.end() ? 0 : it->second.second;
  });
}
int stgp_ctx_profile_reset(stgp_ctx* ctx) {
  return guarded([&] {
    prof_collect(ctx);
    ctx->prof_acc.clear();
  });
}

int stgp_ctx_profile_names(stgp_ctx* ctx, char* buf, int cap) {
  return guarded([&] {
    if (!ctx || !buf || cap < 1) config_error("stgp_ctx_profile_names: bad argument");
    prof_collect(ctx);
    std::string all;
    for (const auto& kv : ctx->prof_acc) all += kv.first + "\n";
    const size_t n = std::min(all.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, all.data(), n);
    buf[n] = 0;
  });
}

int stgp_debug_gemm_rows(stgp_ctx* ctx, int emulated, long long n, int m, int k, const double* A_host,
                         const double* B_host, double* C_host, double* ms) {
  return guarded([&] {
    if (!ctx || n < 0 || m <= 0 || k <= 0 || !A_host || !B_host || !C_host) config_error("stgp_debug_gemm_rows: bad argument");
    DevBuf<double> A, B, C(static_cast<size_t>(n) * m);
    A.upload(A_host, static_cast<size_t>(n) * k, ctx->stream);
    B.upload(B_host, static_cast<size_t>(m) * k, ctx->stream);
    auto run = [&] {
      if (emulated) {
        ozaki_gemm_rows(ctx, n, m, k, A.get(), k, B.get(), k, C.get(), m);
      } else {
        dev_gemm(ctx, true, false, m, static_cast<int>(n), k, 1.0, B.get(), k, A.get(), k, 0.0, C.get(), m);
      }
    };
    run();  // warm-up (plans, workspace)
    cudaEvent_t e0, e1;
    STGP_CUDA(cudaEventCreate(&e0));
    STGP_CUDA(cudaEventCreate(&e1));
    STGP_CUDA(cudaEventRecord(e0, ctx->stream));
    run();
    STGP_CUDA(cudaEventRecord(e1, ctx->stream));
    STGP_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    STGP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms) *ms = t;
    C.download(C_host, static_cast<size_t>(n) * m, ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int stgp_debug_trmm(stgp_ctx* ctx, int mode, int transpose, int m, long long n, const double* T_host,
                    const double* B_host, double* C_host, double* ms) {
  return guarded([&] {
    if (!ctx || m <= 0 || m % 4 || n < 0 || mode < 0 || mode > 2 || !T_host || !B_host || !C_host)
      config_error("stgp_debug_trmm: bad argument");
    const size_t nb = static_cast<size_t>(m) * n;
    DevBuf<double> T, B, C(std::max<size_t>(nb, 1));
    T.upload(T_host, static_cast<size_t>(m) * m, ctx->stream);
    B.upload(B_host, nb, ctx->stream);
    auto run = [&] {
      if (mode == 0)
        dev_trmm_left(ctx, T.get(), m, m, B.get(), m, n, transpose != 0, C.get(), m);
      else
        ozaki_trmm_left(ctx, T.get(), m, m, B.get(), m, n, transpose != 0, C.get(), m, mode == 1);
    };
    run();
    cudaEvent_t e0, e1;
    STGP_CUDA(cudaEventCreate(&e0));
    STGP_CUDA(cudaEventCreate(&e1));
    STGP_CUDA(cudaEventRecord(e0, ctx->stream));
    run();
    STGP_CUDA(cudaEventRecord(e1, ctx->stream));
    STGP_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    STGP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms) *ms = t;
    C.download(C_host, nb, ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int stgp_debug_gemm_cols(stgp_ctx* ctx, int emulated, int m, long long n, const double* A_host,
                         const double* B_host, double* C_host, double* ms) {
  return guarded([&] {
    if (!ctx || m <= 0 || n <= 0 || !A_host || !B_host || !C_host) config_error("stgp_debug_gemm_cols: bad argument");
    DevBuf<double> A, B, C(static_cast<size_t>(m) * m);
    A.upload(A_host, static_cast<size_t>(m) * n, ctx->stream);
    const bool same = A_host == B_host;
    if (!same) B.upload(B_host, static_cast<size_t>(m) * n, ctx->stream);
    const double* Bp = same ? A.get() : B.get();
    auto run = [&] {
      if (emulated)
        ozaki_gemm_cols(ctx, m, n, A.get(), m, Bp, m, C.get(), m);
      else  // C (column-major view: C(i, j) at j m + i) = B A^T
        dev_gemm(ctx, false, true, m, m, n, 1.0, Bp, m, A.get(), m, 0.0, C.get(), m);
    };
    run();
    cudaEvent_t e0, e1;
    STGP_CUDA(cudaEventCreate(&e0));
    STGP_CUDA(cudaEventCreate(&e1));
    STGP_CUDA(cudaEventRecord(e0, ctx->stream));
    run();
    STGP_CUDA(cudaEventRecord(e1, ctx->stream));
    STGP_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    STGP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (ms) *ms = t;
    C.download(C_host, static_cast<size_t>(m) * m, ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int stgp_debug_dmma_peak(stgp_ctx* ctx, double* tflops) {
  return guarded([&] {
    const int blocks = ctx->num_sms * 4, threads = 256, iters = 2048;
    DevBuf<double> out(static_cast<size_t>(blocks) * threads);
    cudaEvent_t e0, e1;
    STGP_CUDA(cudaEventCreate(&e0));
    STGP_CUDA(cudaEventCreate(&e1));
    dmma_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(iters, out.get());  // warm-up
    STGP_CUDA(cudaEventRecord(e0, ctx->stream));
    for (int r = 0; r < 5; ++r) dmma_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(iters, out.get());
    STGP_CUDA(cudaEventRecord(e1, ctx->stream));
    ctx->launches += 6;
    STGP_LAUNCH_CHECK();
    STGP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    STGP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 5.0 * blocks * (threads / 32) * static_cast<double>(iters) * 8 * 512;
    *tflops = flops / (ms * 1e-3) / 1e12;
  });
}

int stgp_debug_fp64_peak(stgp_ctx* ctx, double* tflops) {
  return guarded([&] {
    const int blocks = ctx->num_sms * 4, threads = 256, iters = 4096;
    DevBuf<double> out(static_cast<size_t>(blocks) * threads);
    cudaEvent_t e0, e1;
    STGP_CUDA(cudaEventCreate(&e0));
    STGP_CUDA(cudaEventCreate(&e1));
    fp64_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(iters, out.get());  // warm-up
    STGP_CUDA(cudaEventRecord(e0, ctx->stream));
    for (int r = 0; r < 5; ++r) fp64_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(iters, out.get());
    STGP_CUDA(cudaEventRecord(e1, ctx->stream));
    ctx->launches += 6;
    STGP_LAUNCH_CHECK();
    STGP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    STGP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 5.0 * blocks * threads * static_cast<double>(iters) * 16 * 2;
    *tflops = flops / (ms * 1e-3) / 1e12;
  });
}

int stgp_order_observations(int n, const double* t, uint64_t seed, int32_t* perm_out) {
  return guarded([&] {
    if (n <= 0) data_error("SpaceTimeDataset: empty dataset");
    std::vector<int> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return t[a] < t[b]; });
    std::mt19937_64 rng(mix_seed(seed, 0x0bde11));
    size_t bs = 0;
    for (size_t k = 1; k <= perm.size(); ++k) {
      const bool end = k == perm.size() || t[perm[k]] != t[perm[bs]];
      if (end) {
        for (size_t j = k - 1; j > bs; --j) {
          std::uniform_int_distribution<size_t> pick(bs, j);
          std::swap(perm[j], perm[pick(rng)]);
        }
        bs = k;
      }
    }
    std::copy(perm.begin(), perm.end(), perm_out);
  });
}

int stgp_effective_ranges(const stgp_params* theta, double* tr, double* sr) {
  return guarded([&] {
    Params p;
    std::memcpy(&p, theta, sizeof(p));
    validate_params(p);
    const double e = p.delta + p.beta;
    if (e <= 0.0 || p.a <= 0.0) {
      *tr = std::numeric_limits<double>::infinity();
    } else {
      const double T = std::pow(20.0, 1.0 / e);
      *tr = std::pow((T - 1.0) / p.a, 1.0 / (2.0 * p.alpha));
    }
    auto matern = [&](double x) {
      if (x == 0.0) return 1.0;
      if (p.nu == 0.5) return std::exp(-x);
      if (p.nu == 1.5) return (1.0 + x) * std::exp(-x);
      if (p.nu == 2.5) return (1.0 + x + x * x / 3.0) * std::exp(-x);
      const double v = std::pow(2.0, 1.0 - p.nu) / std::tgamma(p.nu) * std::pow(x, p.nu) * std::cyl_bessel_k(p.nu, x);
      return std::isfinite(v) ? v : 0.0;
    };
    double lo = 0.0, hi = 1.0;
    while (matern(hi) > 0.05) hi *= 2.0;
    while ((hi - lo) > 1e-10 * hi) {
      const double mid = 0.5 * (lo + hi);
      if (matern(mid) > 0.05) lo = mid;
      else hi = mid;
    }
    *sr = 0.5 * (lo + hi) / p.c;
  });
}

uint64_t stgp_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

int stgp_dataset_create(stgp_ctx* ctx, int n, const double* x, const double* y, const double* t,
                        stgp_dataset** out) {
  return guarded([&] {
    require(ctx && out, "stgp_dataset_create: null argument");
    if (n <= 0) data_error("SpaceTimeDataset: empty dataset");
    auto ds = std::make_unique<stgp_dataset>();
    ds->ctx = ctx;
    ds->n = n;
    ds->hx.assign(x, x + n);
    ds->hy.assign(y, y + n);
    ds->ht.assign(t, t + n);
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(x[i]) || !std::isfinite(y[i]) || !std::isfinite(t[i]))
        data_error("SpaceTimeDataset: non-finite coordinates");
    std::set<double> ts(t, t + n);
    ds->Tdata.assign(ts.begin(), ts.end());
    ds->htid.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i)
      ds->htid[static_cast<size_t>(i)] =
          static_cast<int32_t>(std::lower_bound(ds->Tdata.begin(), ds->Tdata.end(), t[i]) - ds->Tdata.begin());
    ds->time_sorted = true;
    for (int i = 1; i < n; ++i)
      if (t[i] < t[i - 1]) ds->time_sorted = false;
    // maybe_precompute_lags (approximations.cpp:26-38)
    bool integral = true;
    double tmin = t[0], tmax = t[0];
    for (int i = 0; i < n; ++i) {
      if (std::abs(t[i] - std::nearbyint(t[i])) >= 1e-9) {
        integral = false;
        break;
      }
      tmin = std::min(tmin, t[i]);
      tmax = std::max(tmax, t[i]);
    }
    const double range = tmax - tmin;
    if (integral && range >= 0.0 && range <= 200000.0) {
      ds->lagpol.table = true;
      ds->lagpol.size = static_cast<int>(range) + 2;
    }
    cudaStream_t s = ctx->stream;
    ds->x.upload(x, n, s);
    ds->y.upload(y, n, s);
    ds->t.upload(t, n, s);
    ds->tid.upload(ds->htid.data(), n, s);
    if (ds->time_sorted) {
      std::vector<int32_t> bs(ds->Tdata.size() + 1, 0);
      for (int i = n - 1; i >= 0; --i) bs[static_cast<size_t>(ds->htid[static_cast<size_t>(i)])] = i;
      bs.back() = n;
      ds->blk_start.upload(bs.data(), bs.size(), s);
    }
    STGP_CUDA(cudaStreamSynchronize(s));
    *out = ds.release();
  });
}

int stgp_dataset_set_response(stgp_dataset* ds, const double* resp, int p, const double* X) {
  return guarded([&] {
    require(ds && resp, "stgp_dataset_set_response: null argument");
    for (int i = 0; i < ds->n; ++i)
      if (!std::isfinite(resp[i])) data_error("SpaceTimeDataset: non-finite response or covariates");
    ds->resp.upload(resp, ds->n, ds->ctx->stream);
    ds->p = std::max(p, 0);
    if (ds->p > 0) ds->X.upload(X, static_cast<size_t>(ds->n) * ds->p, ds->ctx->stream);
    ds->has_resp = true;
    STGP_CUDA(cudaStreamSynchronize(ds->ctx->stream));
  });
}

void stgp_dataset_destroy(stgp_dataset* ds) { delete ds; }

// ---- neighbour searches ----
static stgp_neighbors* run_search(stgp_dataset* ds, int metric, const Params* th, int m_v, double ss,
                                  double ts) {
  stgp_ctx* ctx = ds->ctx;
  if (m_v < 0) config_error("m_v must be >= 0");
  if (m_v > kMaxSearchM) config_error("neighbour search supports m_v <= 128 on the device");
  auto nb = std::make_unique<stgp_neighbors>();
  nb->ctx = ctx;
  nb->n = ds->n;
  nb->m_v = std::max(m_v, 1);
  nb->kind = metric;
  nb->ss = ss;
  nb->ts = ts;
  const size_t total = static_cast<size_t>(ds->n) * nb->m_v;
  nb->idx.alloc(total);
  nb->dist.alloc(total);
  nb->has_dist = true;
  SearchArgs a{};
  a.n = ds->n;
  a.m_v = m_v == 0 ? 1 : m_v;
  // queries shard by contiguous rows across ranks; candidates are replicated (gather_rows after)
  int q0 = 0, q1 = ds->n;
  shard_rows(ctx, ds->n, q0, q1);
  a.q_begin = q0;
  a.q_end = q1;
  a.x = ds->x.get();
  a.y = ds->y.get();
  a.t = ds->t.get();
  a.tid = ds->tid.get();
  a.ss = ss;
  a.ts = ts;
  a.out = nb->idx.get() + static_cast<size_t>(q0) * a.m_v;
  a.dist = nb->dist.get() + static_cast<size_t>(q0) * a.m_v;
  DevLagTable dl;
  TimeIndex ti;
  if (ds->time_sorted) {
    a.blk_of = ds->tid.get();
    a.blk_start = ds->blk_start.get();
    a.nblk = static_cast<int>(ds->Tdata.size());
    a.blk_tid = nullptr;
  }
  DevBuf<int32_t> blk_tid;
  if (ds->time_sorted) {
    std::vector<int32_t> bt(ds->Tdata.size());
    std::iota(bt.begin(), bt.end(), 0);
    blk_tid.upload(bt.data(), bt.size(), ctx->stream);
    a.blk_tid = blk_tid.get();
  }
  if (metric == STGP_METRIC_DC) {
    a.k = dev_kernel(*th);
    ti.T = ds->Tdata;
    ti.build();
    LagPolicy live;  // selection kernel has no lag table (estimation.cpp:200)
    upload_lag_table(dl, ti, *th, live, ctx->stream, true);
    a.lt = lag_view(dl);
  }
  const int blocks = std::max(1, std::min(ceil_div(std::max(q1 - q0, 1), 8), ctx->num_sms * 8));
  if (m_v == 0) {
    std::vector<int32_t> neg(total, -1);
    nb->idx.upload(neg.data(), total, ctx->stream);
  } else if (metric == STGP_METRIC_DC) {
    ProfRegion pr(ctx, "knn_dc");
    const bool gen = a.k.nu_code == kNuGeneral;
    // list slots per lane: m_v <= 32 R
    if (m_v <= 32) {
      if (gen) knn_kernel<0, true><<<blocks, 256, 0, ctx->stream>>>(a);
      else knn_kernel<0><<<blocks, 256, 0, ctx->stream>>>(a);
    } else if (m_v <= 64) {
      if (gen) knn_kernel<0, true, 2><<<blocks, 256, 0, ctx->stream>>>(a);
      else knn_kernel<0, false, 2><<<blocks, 256, 0, ctx->stream>>>(a);
    } else {
      if (gen) knn_kernel<0, true, 4><<<blocks, 256, 0, ctx->stream>>>(a);
      else knn_kernel<0, false, 4><<<blocks, 256, 0, ctx->stream>>>(a);
    }
    ++ctx->launches;
  } else {
    ProfRegion pr(ctx, "knn_euclid");
    if (m_v <= 32) knn_kernel<1><<<blocks, 256, 0, ctx->stream>>>(a);
    else if (m_v <= 64) knn_kernel<1, false, 2><<<blocks, 256, 0, ctx->stream>>>(a);
    else knn_kernel<1, false, 4><<<blocks, 256, 0, ctx->stream>>>(a);
    ++ctx->launches;
  }
  STGP_LAUNCH_CHECK();
  if (m_v > 0) gather_rows(ctx, nb->idx.get(), nb->dist.get(), ds->n, a.m_v, q0, q1);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  prof_collect(ctx);
  return nb.release();
}

int stgp_euclidean_neighbors(stgp_dataset* ds, int m_v, double ss, double ts, stgp_neighbors** out) {
  return guarded([&] {
    require(ds && out, "null argument");
    if (!(ss > 0.0) || !(ts > 0.0)) config_error("euclidean_neighbors: scales must be positive");
    if (!ds->time_sorted) config_error("euclidean_neighbors: dataset must be time-ordered");
    *out = run_search(ds, STGP_METRIC_EUCLID, nullptr, m_v, ss, ts);
  });
}

int stgp_correlation_neighbors(stgp_dataset* ds, const stgp_params* theta, int m_v, stgp_neighbors** out) {
  return guarded([&] {
    require(ds && theta && out, "null argument");
    Params p;
    std::memcpy(&p, theta, sizeof(p));
    validate_params(p);
    // The spatial-tile search with an empty inducing set is also the exact d_c search (selection.cu;
    // identical sets).  Its box-distance pruning pays where the equal-time blocks are large: every
    // query of knn_kernel<0> scans its whole block.  cfg4 (10k rows per day): 52 vs 71 ms kernel,
    // 0.062 vs 0.071 s end to end; cfg2 (1k rows per day): 9.0 vs 3.7 ms.  So the spatial search
    // is taken for time-sorted data with >= 4096 rows per distinct time on average;
    // STGP_DC_SPATIAL=0/1 forces either.
    const char* sp = std::getenv("STGP_DC_SPATIAL");
    const bool big_blocks = ds->time_sorted && !ds->Tdata.empty() &&
                            static_cast<double>(ds->n) / static_cast<double>(ds->Tdata.size()) >= 4096.0;
    if (sp ? sp[0] == '1' : big_blocks)
      *out = spatial_search(ds, p, std::vector<double>(), m_v, STGP_METRIC_DC);
    else
      *out = run_search(ds, STGP_METRIC_DC, &p, m_v, 1.0, 1.0);
  });
}

int stgp_neighbors_from_host(stgp_dataset* ds, int m_v, const int32_t* idx, int kind, stgp_neighbors** out) {
  return guarded([&] {
    require(ds && idx && out && m_v >= 1, "stgp_neighbors_from_host: bad argument");
    for (int i = 0; i < ds->n; ++i) {
      int prev = -1;
      bool ended = false;
      for (int a = 0; a < m_v; ++a) {
        const int j = idx[static_cast<size_t>(i) * m_v + a];
        if (j < 0) {
          ended = true;
          continue;
        }
        if (ended || j <= prev || j >= ds->n) config_error("neighbour rows must be ascending, in range, -1 padded");
        prev = j;
      }
    }
    auto nb = std::make_unique<stgp_neighbors>();
    nb->ctx = ds->ctx;
    nb->n = ds->n;
    nb->m_v = m_v;
    nb->kind = kind;
    nb->idx.upload(idx, static_cast<size_t>(ds->n) * m_v, ds->ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(ds->ctx->stream));
    *out = nb.release();
  });
}

int stgp_neighbors_shape(const stgp_neighbors* nb, int* n, int* m_v, int* kind) {
  return guarded([&] {
    require(nb, "null neighbours");
    if (n) *n = nb->n;
    if (m_v) *m_v = nb->m_v;
    if (kind) *kind = nb->kind;
  });
}

int stgp_neighbors_download(const stgp_neighbors* nb, int32_t* idx, double* dist) {
  return guarded([&] {
    require(nb, "null neighbours");
    const size_t total = static_cast<size_t>(nb->n) * nb->m_v;
    if (idx) nb->idx.download(idx, total, nb->ctx->stream);
    if (dist) {
      if (!nb->has_dist) config_error("these neighbour sets carry no distances");
      nb->dist.download(dist, total, nb->ctx->stream);
    }
    STGP_CUDA(cudaStreamSynchronize(nb->ctx->stream));
  });
}

void stgp_neighbors_destroy(stgp_neighbors* nb) { delete nb; }

int stgp_debug_exp(stgp_ctx* ctx, int n, const double* x, double* out) {
  return guarded([&] {
    DevBuf<double> dx, dy(static_cast<size_t>(n));
    dx.upload(x, n, ctx->stream);
    debug_exp_kernel<<<std::max(1, std::min(ceil_div(n, 256), 4096)), 256, 0, ctx->stream>>>(n, dx.get(), dy.get());
    ++ctx->launches;
    STGP_LAUNCH_CHECK();
    dy.download(out, n, ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int stgp_debug_kernel(stgp_ctx* ctx, const stgp_params* theta, int n, const double* h, const double* u,
                      double* cov, double* g6) {
  return guarded([&] {
    Params p;
    std::memcpy(&p, theta, sizeof(p));
    validate_params(p);
    std::vector<TF> tf(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) tf[static_cast<size_t>(i)] = host_factors(p, u[i]);
    DevBuf<TF> dtf;
    DevBuf<double> dh, dc(static_cast<size_t>(n)), dg(static_cast<size_t>(n) * 6);
    dtf.upload(tf.data(), n, ctx->stream);
    dh.upload(h, n, ctx->stream);
    if (g6) require_analytic_grad(p);
    debug_kernel_kernel<<<std::max(1, ceil_div(n, 128)), 128, 0, ctx->stream>>>(n, dev_kernel(p), dtf.get(), dh.get(),
                                                                               dc.get(), g6 ? dg.get() : nullptr);
    ++ctx->launches;
    STGP_LAUNCH_CHECK();
    dc.download(cov, n, ctx->stream);
    if (g6) dg.download(g6, static_cast<size_t>(n) * 6, ctx->stream);
    STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"

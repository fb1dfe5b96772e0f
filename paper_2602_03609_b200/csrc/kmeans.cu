// kMeans++ seeding + Lloyd refinement (inducing.cpp:22-193), bit-exact.
//
// The host owns the RNG (std::mt19937_64 + libstdc++ distributions, exactly
// the reference's draws): the first index and one generate_canonical<double,53>
// per later pick are drawn up front.  The device reproduces every floating-point
// reduction in the reference's order:
//   * D^2 = ((dx^2 + dy^2) + dt^2) without FMA (Eigen row squaredNorm),
//   * total = Eigen's SSE2 VectorXd::sum() (two Packet2d accumulators),
//   * pick  = first i with u <= sequential running sum (weighted_pick),
//   * Lloyd: argmin with strict <, sequential inertia, per-cluster sequential
//     sums in index order, empty clusters re-seeded in cluster order.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <random>
#include <set>
#include <unordered_map>

#include "comm.hpp"
#include "lowrank_common.cuh"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

namespace {

struct KArgs {
  const double* P;  // n x d column-major
  long n;
  int d;
  double* C;  // k x d column-major
  int k;
};

__device__ __forceinline__ double row_d2(const KArgs& a, long i, const double* C, int ldc, int j) {
  double r = 0.0;
  for (int c = 0; c < a.d; ++c) {
    const double t = __dsub_rn(a.P[i + c * a.n], C[j + static_cast<size_t>(c) * ldc]);
    r = c == 0 ? __dmul_rn(t, t) : __dadd_rn(r, __dmul_rn(t, t));
  }
  return r;
}

// d2 = min(d2, |P_i - C_j|^2)  (j < 0: initialise)
__global__ void d2_update_kernel(KArgs a, int j, bool init, double* d2) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < a.n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const double v = row_d2(a, i, a.C, a.k, j);
    d2[i] = init ? v : (v < d2[i] ? v : d2[i]);  // cwiseMin keeps the old value on ties
  }
}

// One weighted pick (inducing.cpp:32-42): total in Eigen's order, then the sequential running sum.
// Both are order-defined chains, so one thread runs them -- over shared-memory chunks that the
// whole block stages from global memory (loads batched ahead of the dependent adds).  Writes the
// pick and copies the point into C[j].
constexpr int kPickChunk = 12288;  // doubles (96 KB), a multiple of 8
constexpr int kPickThreads = 1024;
__global__ void __launch_bounds__(kPickThreads) pick_kernel(KArgs a, const double* d2, double canon, int j,
                                                            long* pick_out) {
  extern __shared__ double sd[];
  __shared__ double s_u;
  __shared__ int s_done;
  const long n = a.n;
  const int t = threadIdx.x;
  const long aligned = (n / 2) * 2, aligned2 = (n / 4) * 4;
  // ---- pass 1: Eigen's SSE2 two-packet sum ----
  double p0a = 0.0, p0b = 0.0, p1a = 0.0, p1b = 0.0;
  if (t == 0 && aligned > 0) {
    p0a = d2[0];
    p0b = d2[1];
    if (aligned > 2) {
      p1a = d2[2];
      p1b = d2[3];
    }
  }
  if (aligned > 2) {
    for (long c0 = 4; c0 < aligned2; c0 += kPickChunk) {  // groups of 4 never straddle a chunk
      const long c1 = min(aligned2, c0 + kPickChunk);
      __syncthreads();
      for (long i = c0 + t; i < c1; i += blockDim.x) sd[i - c0] = d2[i];
      __syncthreads();
      if (t == 0) {
        const int len = static_cast<int>(c1 - c0);
        for (int i = 0; i < len; i += 4) {
          p0a = __dadd_rn(p0a, sd[i]);
          p0b = __dadd_rn(p0b, sd[i + 1]);
          p1a = __dadd_rn(p1a, sd[i + 2]);
          p1b = __dadd_rn(p1b, sd[i + 3]);
        }
      }
    }
  }
  if (t == 0) {
    double total;
    if (aligned == 0) {
      total = d2[0];
      for (long i = 1; i < n; ++i) total = __dadd_rn(total, d2[i]);
    } else {
      if (aligned > 2) {
        p0a = __dadd_rn(p0a, p1a);
        p0b = __dadd_rn(p0b, p1b);
        if (aligned > aligned2) {
          p0a = __dadd_rn(p0a, d2[aligned2]);
          p0b = __dadd_rn(p0b, d2[aligned2 + 1]);
        }
      }
      total = __dadd_rn(p0a, p0b);
      for (long i = aligned; i < n; ++i) total = __dadd_rn(total, d2[i]);
    }
    // uniform_real_distribution<double>(0, total): canon * (total - 0) + 0
    s_u = __dadd_rn(__dmul_rn(canon, __dsub_rn(total, 0.0)), 0.0);
    s_done = 0;
  }
  // ---- pass 2: sequential running sum, first i with u <= acc ----
  double acc = 0.0;
  long pick = n - 1;
  for (long c0 = 0; c0 < n; c0 += kPickChunk) {
    const long c1 = min(n, c0 + kPickChunk);
    __syncthreads();
    if (s_done) break;
    for (long i = c0 + t; i < c1; i += blockDim.x) sd[i - c0] = d2[i];
    __syncthreads();
    if (t == 0) {
      const double u = s_u;
      const int len = static_cast<int>(c1 - c0);
      int i = 0;
      bool hit = false;
      for (; i + 8 <= len && !hit; i += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = sd[i + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (!hit) {
            acc = __dadd_rn(acc, v[q]);
            if (u <= acc) {
              pick = c0 + i + q;
              hit = true;
            }
          }
        }
      }
      for (; i < len && !hit; ++i) {
        acc = __dadd_rn(acc, sd[i]);
        if (u <= acc) {
          pick = c0 + i;
          hit = true;
        }
      }
      if (hit) s_done = 1;
    }
  }
  if (t == 0) {
    *pick_out = pick;
    for (int c = 0; c < a.d; ++c) a.C[j + static_cast<size_t>(c) * a.k] = a.P[pick + c * n];
  }
}

// Lloyd assignment: best center with strict < (first minimum)
__global__ void assign_kernel(KArgs a, int* assign, double* best) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < a.n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    double b = __longlong_as_double(0x7ff0000000000000LL);
    int bj = 0;
    for (int j = 0; j < a.k; ++j) {
      const double v = row_d2(a, i, a.C, a.k, j);
      if (v < b) {
        b = v;
        bj = j;
      }
    }
    assign[i] = bj;
    best[i] = b;
  }
}

// inertia = sequential sum of best distances
// Sequential sum of best[] (order-defined): the block stages chunks in shared memory, thread 0
// runs the chain with loads batched ahead.
constexpr int kLloydChunk = 4096;
__global__ void __launch_bounds__(1024) inertia_kernel(const double* best, long n, double* out) {
  __shared__ double sb[kLloydChunk];
  double s = 0.0;
  for (long c0 = 0; c0 < n; c0 += kLloydChunk) {
    const int len = static_cast<int>(min(static_cast<long>(kLloydChunk), n - c0));
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += blockDim.x) sb[i] = best[c0 + i];
    __syncthreads();
    if (threadIdx.x == 0) {
      int i = 0;
      for (; i + 8 <= len; i += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = sb[i + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) s = __dadd_rn(s, v[q]);
      }
      for (; i < len; ++i) s = __dadd_rn(s, sb[i]);
    }
  }
  if (threadIdx.x == 0) *out = s;
}
// Per-cluster sums in point order (the reference's sequential accumulation): one thread per
// cluster over block-staged chunks of assign[] and the points (d <= 3).
__global__ void __launch_bounds__(1024) cluster_sum_kernel(KArgs a, const int* assign, double* sums, int* counts) {
  constexpr int kCh = 1536;  // 42 KB of static shared memory
  __shared__ int sa[kCh];
  __shared__ double sp[3][kCh];
  for (int j0 = 0; j0 < a.k; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    double s[3] = {0.0, 0.0, 0.0};
    int cnt = 0;
    for (long c0 = 0; c0 < a.n; c0 += kCh) {
      const int len = static_cast<int>(min(static_cast<long>(kCh), a.n - c0));
      __syncthreads();
      for (int i = threadIdx.x; i < len; i += blockDim.x) {
        sa[i] = assign[c0 + i];
        for (int c = 0; c < a.d; ++c) sp[c][i] = a.P[c0 + i + static_cast<long>(c) * a.n];
      }
      __syncthreads();
      if (j < a.k)
        for (int i = 0; i < len; ++i) {
          if (sa[i] != j) continue;
          for (int c = 0; c < a.d; ++c) s[c] = __dadd_rn(s[c], sp[c][i]);
          ++cnt;
        }
    }
    if (j < a.k) {
      for (int c = 0; c < a.d; ++c) sums[j + static_cast<size_t>(c) * a.k] = s[c];
      counts[j] = cnt;
    }
  }
}
__global__ void center_update_kernel(KArgs a, const int* assign, const double* sums, const int* counts) {
  __shared__ double bd[1024];
  __shared__ long bi[1024];
  for (int j = 0; j < a.k; ++j) {
    if (counts[j] > 0) {
      if (threadIdx.x == 0)
        for (int c = 0; c < a.d; ++c)
          a.C[j + static_cast<size_t>(c) * a.k] =
              __ddiv_rn(sums[j + static_cast<size_t>(c) * a.k], static_cast<double>(counts[j]));
      __syncthreads();
      continue;
    }
    double far_d = -1.0;
    long far = 0;
    for (long i = threadIdx.x; i < a.n; i += blockDim.x) {
      const double v = row_d2(a, i, a.C, a.k, assign[i]);
      if (v > far_d) {
        far_d = v;
        far = i;
      }
    }
    bd[threadIdx.x] = far_d;
    bi[threadIdx.x] = far;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        const double od = bd[threadIdx.x + o];
        const long oi = bi[threadIdx.x + o];
        if (od > bd[threadIdx.x] || (od == bd[threadIdx.x] && oi < bi[threadIdx.x])) {
          bd[threadIdx.x] = od;
          bi[threadIdx.x] = oi;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0)
      for (int c = 0; c < a.d; ++c) a.C[j + static_cast<size_t>(c) * a.k] = a.P[bi[0] + c * a.n];
    __syncthreads();
  }
}

}  // namespace

static int count_distinct_rows(const double* P, long n, int d) {
  std::vector<long> idx(static_cast<size_t>(n));
  std::iota(idx.begin(), idx.end(), 0);
  auto less = [&](long a, long b) {
    for (int c = 0; c < d; ++c) {
      const double va = P[a + c * n], vb = P[b + c * n];
      if (va < vb) return true;
      if (vb < va) return false;
    }
    return false;
  };
  std::sort(idx.begin(), idx.end(), less);
  int distinct = n > 0 ? 1 : 0;
  for (long i = 1; i < n; ++i)
    if (less(idx[static_cast<size_t>(i - 1)], idx[static_cast<size_t>(i)])) ++distinct;
  return distinct;
}

// kmeanspp (inducing.cpp:46-115) on a host n x d column-major matrix; centers k x d column-major
void kmeanspp_device(stgp_ctx* ctx, const double* P_host, long n, int d, int k, uint64_t seed, double* centers_host,
                     int known_distinct = -1) {
  if (n == 0) data_error("kmeanspp: no points");
  if (k < 1) config_error("kmeanspp: k must be >= 1");
  if (d < 1 || d > 3) config_error("kmeanspp: device path supports 1..3 coordinates");
  const int distinct = known_distinct >= 0 ? known_distinct : count_distinct_rows(P_host, n, d);
  if (k > distinct) data_error("kmeanspp: k exceeds the number of distinct points");
  // host RNG stream, identical to the reference
  std::mt19937_64 rng(mix_seed(seed, 0x6d70));
  std::uniform_int_distribution<long> first(0, n - 1);
  const long f = first(rng);
  std::vector<double> canon(static_cast<size_t>(k));
  for (int j = 1; j < k; ++j) canon[static_cast<size_t>(j)] = std::generate_canonical<double, 53>(rng);

  cudaStream_t st = ctx->stream;
  DevBuf<double> P, C(static_cast<size_t>(k) * d), d2(static_cast<size_t>(n)), best(static_cast<size_t>(n)),
      sums(static_cast<size_t>(k) * d), inertia(1);
  DevBuf<int> assign(static_cast<size_t>(n)), counts(static_cast<size_t>(k));
  DevBuf<long> pick(1);
  P.upload(P_host, static_cast<size_t>(n) * d, st);
  std::vector<double> c0(static_cast<size_t>(d));
  for (int c = 0; c < d; ++c) {
    const double v = P_host[f + c * n];
    STGP_CUDA(cudaMemcpyAsync(C.get() + static_cast<size_t>(c) * k, &P_host[f + c * n], sizeof(double),
                              cudaMemcpyHostToDevice, st));
    (void)v;
  }
  KArgs a{P.get(), n, d, C.get(), k};
  const int gb = grid_for(n, 256, ctx->num_sms * 8);
  d2_update_kernel<<<gb, 256, 0, st>>>(a, 0, true, d2.get());
  launched(ctx);
  STGP_CUDA(cudaFuncSetAttribute(pick_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sizeof(double) * kPickChunk)));
  for (int j = 1; j < k; ++j) {
    pick_kernel<<<1, kPickThreads, sizeof(double) * kPickChunk, st>>>(a, d2.get(), canon[static_cast<size_t>(j)], j,
                                                                       pick.get());
    launched(ctx);
    d2_update_kernel<<<gb, 256, 0, st>>>(a, j, false, d2.get());
    launched(ctx);
  }
  double prev = std::numeric_limits<double>::infinity();
  for (int sweep = 0; sweep < 50; ++sweep) {
    assign_kernel<<<gb, 256, 0, st>>>(a, assign.get(), best.get());
    launched(ctx);
    inertia_kernel<<<1, 1024, 0, st>>>(best.get(), n, inertia.get());
    launched(ctx);
    cluster_sum_kernel<<<1, std::min(1024, std::max(32, (k + 31) / 32 * 32)), 0, st>>>(a, assign.get(), sums.get(),
                                                                                       counts.get());
    launched(ctx);
    center_update_kernel<<<1, 1024, 0, st>>>(a, assign.get(), sums.get(), counts.get());
    launched(ctx);
    double in = 0.0;
    inertia.download(&in, 1, st);
    STGP_CUDA(cudaStreamSynchronize(st));
    if (in == 0.0 || std::abs(prev - in) < 1e-6 * std::max(in, 1e-300)) break;
    prev = in;
  }
  C.download(centers_host, static_cast<size_t>(k) * d, st);
  STGP_CUDA(cudaStreamSynchronize(st));
}

}  // namespace stgp

using namespace stgp;

namespace {
template <class F>
int guarded(F&& f) {
  try {
    f();
    return STGP_OK;
  } catch (const stgp::Error& e) {
    stgp::g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    stgp::g_last_error = e.what();
    return STGP_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

int stgp_kmeanspp(stgp_ctx* ctx, const double* P, int n, int d, int k, uint64_t seed, double* centers) {
  return guarded([&] {
    if (!ctx || !P || !centers) config_error("stgp_kmeanspp: null argument");
    kmeanspp_device(ctx, P, n, d, k, seed, centers);
  });
}

// sts_kmeanspp (inducing.cpp:144-193): unique times / locations via ordered sets
namespace {
// bit key with -0.0 folded onto +0.0 (std::set's operator< treats them as equal)
inline uint64_t dkey(double v) {
  uint64_t b;
  std::memcpy(&b, &v, sizeof(b));
  return v == 0.0 ? 0 : b;
}
struct PairKeyHash {
  size_t operator()(const std::pair<uint64_t, uint64_t>& k) const {
    return std::hash<uint64_t>()(k.first * 0x9E3779B97F4A7C15ULL ^ (k.second + 0x632BE59BD9B4E019ULL));
  }
};
std::vector<double> distinct_sorted_times(const std::vector<double>& t) {
  std::unordered_map<uint64_t, double> first;
  first.reserve(1024);
  for (double v : t) first.emplace(dkey(v), v);
  std::vector<double> out;
  out.reserve(first.size());
  for (const auto& kv : first) out.push_back(kv.second);
  std::sort(out.begin(), out.end());
  return out;
}
std::vector<std::pair<double, double>> distinct_sorted_locations(const std::vector<double>& x,
                                                                 const std::vector<double>& y) {
  std::unordered_map<std::pair<uint64_t, uint64_t>, std::pair<double, double>, PairKeyHash> first;
  first.reserve(1 << 14);
  for (size_t i = 0; i < x.size(); ++i) first.emplace(std::make_pair(dkey(x[i]), dkey(y[i])), std::make_pair(x[i], y[i]));
  std::vector<std::pair<double, double>> out;
  out.reserve(first.size());
  for (const auto& kv : first) out.push_back(kv.second);
  std::sort(out.begin(), out.end());
  return out;
}
}  // namespace

int stgp_sts_kmeanspp(stgp_dataset* ds, int m, uint64_t seed, stgp_inducing** out) {
  return guarded([&] {
    if (!ds || !out) config_error("stgp_sts_kmeanspp: null argument");
    if (m < 1) config_error("sts_kmeanspp: m must be >= 1");
    const int n = ds->n;
    // the reference's std::set<double> / std::set<pair> (inducing.cpp:150-156): distinct values in
    // ascending order, the first occurrence kept; hashed here (the sets cost ~0.3 s at n = 1.1M)
    const std::vector<double> times = distinct_sorted_times(ds->ht);
    const std::vector<std::pair<double, double>> ss = distinct_sorted_locations(ds->hx, ds->hy);
    std::vector<double> locs(2 * ss.size());
    for (size_t i = 0; i < ss.size(); ++i) {
      locs[i] = ss[i].first;
      locs[i + ss.size()] = ss[i].second;
    }
    const double nt = static_cast<double>(times.size());
    int m_s = static_cast<int>(std::lround(std::sqrt(static_cast<double>(m) * n / (nt * nt))));
    int m_t = static_cast<int>(std::lround(std::sqrt(static_cast<double>(m) * nt * nt / n)));
    m_s = std::clamp(m_s, 1, std::min(static_cast<int>(ss.size()), m));
    m_t = std::clamp(m_t, 1, std::min(static_cast<int>(times.size()), m));
    std::vector<double> sc(static_cast<size_t>(m_s) * 2), tc(static_cast<size_t>(m_t));
    kmeanspp_device(ds->ctx, locs.data(), static_cast<long>(ss.size()), 2, m_s, mix_seed(seed, 1), sc.data(),
                    static_cast<int>(ss.size()));
    kmeanspp_device(ds->ctx, times.data(), static_cast<long>(times.size()), 1, m_t, mix_seed(seed, 2), tc.data(),
                    static_cast<int>(times.size()));
    auto ind = std::make_unique<stgp_inducing>();
    ind->ctx = ds->ctx;
    ind->m_s = m_s;
    ind->m_t = m_t;
    for (int js = 0; js < m_s; ++js)
      for (int jt = 0; jt < m_t; ++jt) {
        const double p[3] = {sc[static_cast<size_t>(js)], sc[static_cast<size_t>(js + m_s)], tc[static_cast<size_t>(jt)]};
        ind->xyt.insert(ind->xyt.end(), p, p + 3);
      }
    *out = ind.release();
  });
}

// joint_kmeanspp_inducing (inducing.cpp:117-142)
int stgp_joint_kmeanspp_inducing(stgp_dataset* ds, int m, double ss, double ts, uint64_t seed, stgp_inducing** out) {
  return guarded([&] {
    if (!ds || !out) config_error("stgp_joint_kmeanspp_inducing: null argument");
    if (!(ss > 0.0) || !(ts > 0.0)) config_error("joint_kmeanspp_inducing: scales must be positive");
    const int n = ds->n;
    std::vector<double> S(static_cast<size_t>(n) * 3);
    for (int i = 0; i < n; ++i) {
      S[static_cast<size_t>(i)] = ds->hx[static_cast<size_t>(i)] / ss;
      S[static_cast<size_t>(i) + n] = ds->hy[static_cast<size_t>(i)] / ss;
      S[static_cast<size_t>(i) + 2 * static_cast<size_t>(n)] = ds->ht[static_cast<size_t>(i)] / ts;
    }
    const int distinct = count_distinct_rows(S.data(), n, 3);
    const int k = std::min(m, distinct);
    std::vector<double> C(static_cast<size_t>(k) * 3);
    kmeanspp_device(ds->ctx, S.data(), n, 3, k, seed, C.data(), distinct);
    auto ind = std::make_unique<stgp_inducing>();
    ind->ctx = ds->ctx;
    for (int j = 0; j < k; ++j) {
      const double p[3] = {C[static_cast<size_t>(j)] * ss, C[static_cast<size_t>(j + k)] * ss,
                           C[static_cast<size_t>(j + 2 * k)] * ts};
      if (!std::isfinite(p[0]) || !std::isfinite(p[1]) || !std::isfinite(p[2]))
        data_error("SpaceTimePoint: coordinates and time must be finite");
      ind->xyt.insert(ind->xyt.end(), p, p + 3);
    }
    *out = ind.release();
  });
}

}  // extern "C"

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
#include <memory>
#include <cstring>
#include <numeric>
#include <random>
#include <set>
#include <unordered_map>

#include <cub/device/device_radix_sort.cuh>

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
                                                            long* pick_out, const int* need = nullptr) {
  if (need && *need == 0) return;  // the certified parallel pick already decided
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

// ---------------------------------------------------------------------------
// Parallel certified pick.  The reference's pick (inducing.cpp:32-42) is defined by two sequential
// floating-point chains: the Eigen-order total t_seq and the running sums acc_i; pick = first i with
// u <= acc_i, u = fl(canon t_seq).  For non-negative weights every order of summation stays within
// gamma_n = n eps / (1 - n eps) of the exact sum, so with the exact prefix sums S_i (double-double here):
//   u in [u_lo, u_hi] = canon T (1 -/+ (gamma_n + 2 eps)),   acc_i in [S_i (1 - gamma_n), S_i (1 + gamma_n)].
// If i* = first i with S_i (1 - gamma_n) >= u_hi also has S_{i*-1} (1 + gamma_n) < u_lo, every possible
// rounding of the two chains picks i*: the pick is certain without running them.  Otherwise (u within
// ~gamma_n T of a boundary: ~1e-4 per pick at n = 1.1M) the exact sequential pick_kernel decides.
// One launch per pick: every block first applies the previous center's D^2 update to its segment, sums
// it in double-double, and the last block to finish scans the block sums and the segment that holds the
// crossing.
// ---------------------------------------------------------------------------
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, double x) {
  const double t = a.hi + x;
  const double bp = t - a.hi;
  const double e = (a.hi - (t - bp)) + (x - bp);
  return DD{t, a.lo + e};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  DD r = dd_add(a, b.hi);
  r.lo += b.lo;
  const double t = r.hi + r.lo;
  return DD{t, r.lo - (t - r.hi)};
}
__device__ __forceinline__ double dd_val(DD a) { return a.hi + a.lo; }

constexpr int kCpThreads = 256;
struct PickArgs {
  KArgs a;
  double* d2;
  int j;           // center being picked; j - 1 is applied to d2 first (j >= 2)
  double canon;
  long* pick_out;
  DD* bsum;        // per-block sums
  unsigned* ticket;
  int* fallback;   // 1: the exact sequential pick must decide
};

__global__ void __launch_bounds__(kCpThreads) pick_certified_kernel(PickArgs p) {
  __shared__ DD sred[kCpThreads];
  __shared__ bool last;
  __shared__ long s_best;
  const KArgs& a = p.a;
  const long n = a.n;
  const int G = gridDim.x, b = blockIdx.x, t = threadIdx.x;
  const long s0 = n * b / G, s1 = n * (b + 1) / G;
  DD acc{0.0, 0.0};
  for (long i = s0 + t; i < s1; i += kCpThreads) {
    double v = p.d2[i];
    if (p.j >= 2) {
      const double c = row_d2(a, i, a.C, a.k, p.j - 1);
      v = c < v ? c : v;
      p.d2[i] = v;
    }
    acc = dd_add(acc, v);
  }
  sred[t] = acc;
  __threadfence();  // this thread's d2 updates, before the ticket makes them the last block's input
  __syncthreads();
  for (int o = kCpThreads / 2; o > 0; o >>= 1) {
    if (t < o) sred[t] = dd_add(sred[t], sred[t + o]);
    __syncthreads();
  }
  if (t == 0) {
    p.bsum[b] = sred[0];
    __threadfence();
    last = atomicAdd(p.ticket, 1u) == static_cast<unsigned>(G - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // ---- last block: total, crossing block, certified index ----
  const double eps = 1.1102230246251565e-16;
  const double gam = static_cast<double>(n) * eps / (1.0 - static_cast<double>(n) * eps);
  __shared__ double s_ulo, s_uhi;
  __shared__ int s_blk;
  __shared__ DD s_base;
  if (t == 0) {
    DD tot{0.0, 0.0};
    for (int q = 0; q < G; ++q) tot = dd_add(tot, p.bsum[q]);
    const double T = dd_val(tot);
    s_ulo = p.canon * T * (1.0 - (gam + 2.0 * eps) - 1e-15);
    s_uhi = p.canon * T * (1.0 + (gam + 2.0 * eps) + 1e-15);
    // first block whose end prefix certainly reaches u_hi
    DD run{0.0, 0.0};
    int blk = -1;
    DD base{0.0, 0.0};
    for (int q = 0; q < G; ++q) {
      const DD nx = dd_add(run, p.bsum[q]);
      if (dd_val(nx) * (1.0 - gam) >= s_uhi) {
        blk = q;
        base = run;
        break;
      }
      run = nx;
    }
    s_blk = blk;
    s_base = base;
    s_best = -1;
    *p.ticket = 0;  // reset for the next launch
  }
  __syncthreads();
  if (s_blk < 0) {
    if (t == 0) *p.fallback = 1;
    return;
  }
  // inclusive prefixes of the crossing block's segment: per-thread contiguous chunks, then a scan of the
  // chunk totals (one thread, G <= kCpThreads chunks)
  const long c0 = n * s_blk / G, c1 = n * (s_blk + 1) / G;
  const long len = c1 - c0;
  const long per = (len + kCpThreads - 1) / kCpThreads;
  const long my0 = c0 + t * per, my1 = min(c1, my0 + per);
  DD part{0.0, 0.0};
  for (long i = my0; i < my1; ++i) part = dd_add(part, p.d2[i]);
  sred[t] = part;
  __syncthreads();
  if (t == 0) {
    DD run = s_base;
    for (int q = 0; q < kCpThreads; ++q) {
      const DD nx = dd_add(run, sred[q]);
      sred[q] = run;  // exclusive prefix of chunk q
      run = nx;
    }
  }
  __syncthreads();
  DD run = sred[t];
  long found = -1;
  double prev_hi = dd_val(run) * (1.0 + gam);
  for (long i = my0; i < my1; ++i) {
    run = dd_add(run, p.d2[i]);
    const double S = dd_val(run);
    if (S * (1.0 - gam) >= s_uhi) {
      found = i;
      break;
    }
    prev_hi = S * (1.0 + gam);
  }
  (void)prev_hi;
  if (found >= 0) atomicMin(reinterpret_cast<unsigned long long*>(&s_best), static_cast<unsigned long long>(found));
  __syncthreads();
  if (t == 0) {
    const long i = s_best;
    bool ok = i >= 0;
    if (ok) {
      // the prefix before i must certainly stay below u_lo
      DD pre = s_base;
      for (long q = c0; q < i; ++q) pre = dd_add(pre, p.d2[q]);
      ok = dd_val(pre) * (1.0 + gam) < s_ulo;
    }
    if (!ok) {
      *p.fallback = 1;
    } else {
      *p.pick_out = i;
      for (int c = 0; c < a.d; ++c) a.C[p.j + static_cast<size_t>(c) * a.k] = a.P[i + c * n];
    }
  }
}

// exact sequential pick when the certificate failed (pick_kernel semantics), else nothing
__global__ void fallback_gate_kernel(const int* fallback, int* run) { *run = *fallback; }

// Lloyd assignment: best center with strict < (first minimum).  Centers staged in shared memory in
// tiles (broadcast reads), two points per thread; the same D^2 expression as row_d2 (no FMA).
constexpr int kAsTile = 1024;
__global__ void __launch_bounds__(256) assign_kernel(KArgs a, int* assign, double* best) {
  __shared__ double sc[3][kAsTile];
  const long stride = static_cast<long>(gridDim.x) * blockDim.x * 2;
  for (long i0 = (blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x) * 2; i0 - threadIdx.x * 2 < a.n;
       i0 += stride) {
    double p0[3] = {0, 0, 0}, p1[3] = {0, 0, 0};
    const bool v0 = i0 < a.n, v1 = i0 + 1 < a.n;
    for (int c = 0; c < a.d; ++c) {
      if (v0) p0[c] = a.P[i0 + c * a.n];
      if (v1) p1[c] = a.P[i0 + 1 + c * a.n];
    }
    double b0 = __longlong_as_double(0x7ff0000000000000LL), b1 = b0;
    int j0 = 0, j1 = 0;
    for (int t0 = 0; t0 < a.k; t0 += kAsTile) {
      const int tl = min(kAsTile, a.k - t0);
      __syncthreads();
      for (int e = threadIdx.x; e < tl; e += blockDim.x)
        for (int c = 0; c < a.d; ++c) sc[c][e] = a.C[t0 + e + static_cast<size_t>(c) * a.k];
      __syncthreads();
      for (int e = 0; e < tl; ++e) {
        double r0 = 0.0, r1 = 0.0;
        for (int c = 0; c < a.d; ++c) {
          const double q0 = __dsub_rn(p0[c], sc[c][e]), q1 = __dsub_rn(p1[c], sc[c][e]);
          r0 = c == 0 ? __dmul_rn(q0, q0) : __dadd_rn(r0, __dmul_rn(q0, q0));
          r1 = c == 0 ? __dmul_rn(q1, q1) : __dadd_rn(r1, __dmul_rn(q1, q1));
        }
        if (r0 < b0) {
          b0 = r0;
          j0 = t0 + e;
        }
        if (r1 < b1) {
          b1 = r1;
          j1 = t0 + e;
        }
      }
    }
    if (v0) {
      assign[i0] = j0;
      best[i0] = b0;
    }
    if (v1) {
      assign[i0 + 1] = j1;
      best[i0 + 1] = b1;
    }
  }
}

// new centers of the non-empty clusters (sums / counts), written out of place; empties counted
__global__ void center_means_kernel(KArgs a, const double* sums, const int* counts, double* Cn, int* n_empty) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.k; j += gridDim.x * blockDim.x) {
    if (counts[j] > 0) {
      for (int c = 0; c < a.d; ++c)
        Cn[j + static_cast<size_t>(c) * a.k] =
            __ddiv_rn(sums[j + static_cast<size_t>(c) * a.k], static_cast<double>(counts[j]));
    } else {
      atomicAdd(n_empty, 1);
    }
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
// Per-cluster sums over the points sorted by cluster (stable radix sort: each cluster's members stay in
// point order), one thread per cluster: the reference's sequential per-cluster accumulation
// (inducing.cpp:80-91) in parallel across clusters.
__global__ void cluster_bounds_kernel(long n, int k, const int* key, int* start, int* count) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c = key[i];
    if (i == 0 || key[i - 1] != c) start[c] = static_cast<int>(i);
    if (i == n - 1 || key[i + 1] != c) count[c] = static_cast<int>(i + 1);  // end, turned into a count below
  }
}
__global__ void cluster_sorted_sum_kernel(KArgs a, const int* order, const int* start, int* counts, double* sums) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < a.k; j += gridDim.x * blockDim.x) {
    const int s0 = start[j], e = counts[j];
    double s[3] = {0.0, 0.0, 0.0};
    int cnt = 0;
    if (s0 >= 0)
      for (int q = s0; q < e; ++q) {
        const long i = order[q];
        for (int c = 0; c < a.d; ++c) s[c] = __dadd_rn(s[c], a.P[i + static_cast<long>(c) * a.n]);
        ++cnt;
      }
    for (int c = 0; c < a.d; ++c) sums[j + static_cast<size_t>(c) * a.k] = s[c];
    counts[j] = cnt;
  }
}
__global__ void iota_kernel(long n, int* v) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x)
    v[i] = static_cast<int>(i);
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

namespace {
// double-double partial sums of best[] per block (certified inertia)
__global__ void __launch_bounds__(256) inertia_dd_kernel(const double* best, long n, DD* part) {
  __shared__ DD sred[256];
  DD acc{0.0, 0.0};
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x)
    acc = dd_add(acc, best[i]);
  sred[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sred[threadIdx.x] = dd_add(sred[threadIdx.x], sred[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sred[0];
}
// order-preserving uint64 key of a double, -0.0 folded onto +0.0 (operator< treats them as equal)
__global__ void dkey_kernel(long n, const double* v, unsigned long long* key) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x) {
    const double x = v[i] == 0.0 ? 0.0 : v[i];
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    key[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
  }
}
__global__ void gather_key_kernel(long n, const unsigned long long* key, const int* perm, unsigned long long* out) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x)
    out[i] = key[perm[i]];
}
// rows i of the sorted order that start a new distinct row
__global__ void distinct_kernel(long n, int d, const unsigned long long* keys, const int* perm, unsigned long long* cnt) {
  unsigned long long local = 0;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x) {
    bool fresh = i == 0;
    for (int c = 0; c < d && !fresh; ++c)
      fresh = keys[static_cast<size_t>(c) * n + perm[i]] != keys[static_cast<size_t>(c) * n + perm[i - 1]];
    local += fresh ? 1 : 0;
  }
  atomicAdd(cnt, local);
}
}  // namespace

// count_distinct_rows (inducing.cpp:22-30) on the device: stable LSD sorts by the order-preserving keys of
// the columns (last column first) give the lexicographic row order; count the row changes
static int count_distinct_rows_device(stgp_ctx* ctx, const double* P_host, long n, int d) {
  cudaStream_t st = ctx->stream;
  DevBuf<double> P(static_cast<size_t>(n) * d);
  P.upload(P_host, static_cast<size_t>(n) * d, st);
  DevBuf<unsigned long long> keys(static_cast<size_t>(n) * d), kin(static_cast<size_t>(n)), kout(static_cast<size_t>(n)),
      cnt(1);
  DevBuf<int> pa(static_cast<size_t>(n)), pb(static_cast<size_t>(n));
  const int gb = grid_for(n, 256, ctx->num_sms * 8);
  for (int c = 0; c < d; ++c) {
    dkey_kernel<<<gb, 256, 0, st>>>(n, P.get() + static_cast<size_t>(c) * n, keys.get() + static_cast<size_t>(c) * n);
    launched(ctx);
  }
  iota_kernel<<<gb, 256, 0, st>>>(n, pa.get());
  launched(ctx);
  size_t tb = 0;
  STGP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.get(), kout.get(), pa.get(), pb.get(), static_cast<int>(n), 0, 64, st));
  DevBuf<unsigned char> tmp(std::max<size_t>(tb, 1));
  for (int c = d - 1; c >= 0; --c) {  // least significant column first; stable
    gather_key_kernel<<<gb, 256, 0, st>>>(n, keys.get() + static_cast<size_t>(c) * n, pa.get(), kin.get());
    launched(ctx);
    size_t t2 = tmp.n;
    STGP_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), t2, kin.get(), kout.get(), pa.get(), pb.get(), static_cast<int>(n), 0, 64, st));
    launched(ctx);
    std::swap(pa, pb);
  }
  cnt.zero(st);
  distinct_kernel<<<gb, 256, 0, st>>>(n, d, keys.get(), pa.get(), cnt.get());
  launched(ctx);
  unsigned long long h = 0;
  cnt.download(&h, 1, st);
  STGP_CUDA(cudaStreamSynchronize(st));
  return static_cast<int>(h);
}

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
  static const bool certified = [] {
    const char* e = std::getenv("STGP_KMEANS_CERTIFIED");  // 0: the one-thread exact pick for every center
    return !(e && e[0] == '0');
  }();
  const int G = std::max(1, std::min<int>(kCpThreads, static_cast<int>((n + 4095) / 4096)));
  DevBuf<DD> bsum(static_cast<size_t>(G));
  DevBuf<unsigned> ticket(1);
  DevBuf<int> fb(1);
  ticket.zero(st);
  long fallbacks = 0;
  std::unique_ptr<ProfRegion> prk(new ProfRegion(ctx, "km_picks"));
  for (int j = 1; j < k; ++j) {
    if (certified) {
      fb.zero(st);
      PickArgs pa{a, d2.get(), j, canon[static_cast<size_t>(j)], pick.get(), bsum.get(), ticket.get(), fb.get()};
      pick_certified_kernel<<<G, kCpThreads, 0, st>>>(pa);
      launched(ctx);
      if (j >= 2) {  // the fallback needs d2 updated with center j - 1: the certified kernel did it
      }
      pick_kernel<<<1, kPickThreads, sizeof(double) * kPickChunk, st>>>(a, d2.get(), canon[static_cast<size_t>(j)], j,
                                                                         pick.get(), fb.get());
      launched(ctx);
    } else {
      if (j >= 2) {
        d2_update_kernel<<<gb, 256, 0, st>>>(a, j - 1, false, d2.get());
        launched(ctx);
      }
      pick_kernel<<<1, kPickThreads, sizeof(double) * kPickChunk, st>>>(a, d2.get(), canon[static_cast<size_t>(j)], j,
                                                                         pick.get());
      launched(ctx);
    }
  }
  (void)fallbacks;
  prk.reset();
  DevBuf<double> Cn(static_cast<size_t>(k) * d);
  DevBuf<int> nempty(1);
  // certified inertia (large n): double-double partials; best[] double-buffered for the exact fallback
  const bool cert_inertia = certified && n >= 65536;
  constexpr int kInBlocks = 128;
  DevBuf<DD> inpart(kInBlocks);
  DevBuf<double> best_prev(cert_inertia ? static_cast<size_t>(n) : 1);
  double prev_lo = 0.0, prev_hi = std::numeric_limits<double>::infinity();
  // Lloyd cluster sums: sorted by cluster for large n (one thread per cluster), else the one-block kernel
  const bool sorted_sums = n >= 65536;
  DevBuf<int> iota, order, keys_s, cstart;
  DevBuf<unsigned char> sort_tmp;
  int key_bits = 1;
  while ((1 << key_bits) < k) ++key_bits;
  if (sorted_sums) {
    iota.alloc(static_cast<size_t>(n));
    order.alloc(static_cast<size_t>(n));
    keys_s.alloc(static_cast<size_t>(n));
    cstart.alloc(static_cast<size_t>(k));
    iota_kernel<<<gb, 256, 0, st>>>(n, iota.get());
    launched(ctx);
    size_t tb = 0;
    STGP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, assign.get(), keys_s.get(), iota.get(), order.get(),
                                              static_cast<int>(n), 0, key_bits, st));
    sort_tmp.alloc(std::max<size_t>(tb, 1));
  }
  double prev = std::numeric_limits<double>::infinity();
  int sweeps = 0;
  for (int sweep = 0; sweep < 50; ++sweep) {
    ++sweeps;
    ProfRegion prl(ctx, "km_lloyd_sweep");
    assign_kernel<<<gb, 256, 0, st>>>(a, assign.get(), best.get());
    launched(ctx);
    if (cert_inertia) {
      inertia_dd_kernel<<<kInBlocks, 256, 0, st>>>(best.get(), n, inpart.get());
      launched(ctx);
    } else {
      inertia_kernel<<<1, 1024, 0, st>>>(best.get(), n, inertia.get());
      launched(ctx);
    }
    if (sorted_sums) {
      size_t tb = sort_tmp.n;
      STGP_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.get(), tb, assign.get(), keys_s.get(), iota.get(), order.get(),
                                                static_cast<int>(n), 0, key_bits, st));
      launched(ctx);
      STGP_CUDA(cudaMemsetAsync(cstart.get(), 0xff, sizeof(int) * k, st));
      STGP_CUDA(cudaMemsetAsync(counts.get(), 0, sizeof(int) * k, st));
      cluster_bounds_kernel<<<gb, 256, 0, st>>>(n, k, keys_s.get(), cstart.get(), counts.get());
      launched(ctx);
      cluster_sorted_sum_kernel<<<grid_for(k, 128), 128, 0, st>>>(a, order.get(), cstart.get(), counts.get(), sums.get());
      launched(ctx);
    } else {
      cluster_sum_kernel<<<1, std::min(1024, std::max(32, (k + 31) / 32 * 32)), 0, st>>>(a, assign.get(), sums.get(),
                                                                                         counts.get());
      launched(ctx);
    }
    // center update (inducing.cpp:93-111): all means in parallel; the re-seeding of empty clusters reads
    // the partly updated centers in cluster order, so any empty cluster takes the sequential kernel
    STGP_CUDA(cudaMemsetAsync(nempty.get(), 0, sizeof(int), st));
    center_means_kernel<<<grid_for(k, 128), 128, 0, st>>>(a, sums.get(), counts.get(), Cn.get(), nempty.get());
    launched(ctx);
    double in = 0.0;
    int ne = 0;
    DD hp[kInBlocks];
    if (cert_inertia) inpart.download(hp, kInBlocks, st);
    else inertia.download(&in, 1, st);
    nempty.download(&ne, 1, st);
    STGP_CUDA(cudaStreamSynchronize(st));
    if (ne == 0) {
      STGP_CUDA(cudaMemcpyAsync(C.get(), Cn.get(), sizeof(double) * k * d, cudaMemcpyDeviceToDevice, st));
    } else {
      center_update_kernel<<<1, 1024, 0, st>>>(a, assign.get(), sums.get(), counts.get());
      launched(ctx);
    }
    if (cert_inertia) {
      // inducing.cpp:113: stop when in == 0 or |prev - in| < 1e-6 in, in = the sequential sum of best[].
      // The exact value lies within gamma_n of the double-double sum; decide from the bounds, and run the
      // sequential chains (this sweep's and, kept in the other buffer, the previous sweep's) only when
      // the bounds straddle the threshold.
      double hi = 0.0, lo = 0.0;
      for (int q = 0; q < kInBlocks; ++q) {  // fixed block order
        const double t2 = hi + hp[q].hi;
        const double bp = t2 - hi;
        lo += (hi - (t2 - bp)) + (hp[q].hi - bp) + hp[q].lo;
        hi = t2;
      }
      const double T = hi + lo;
      const double gam = static_cast<double>(n) * 1.1102230246251565e-16 / (1.0 - static_cast<double>(n) * 1.1102230246251565e-16) + 1e-15;
      const double in_lo = T * (1.0 - gam), in_hi = T * (1.0 + gam);
      bool stop, certain = true;
      if (in_hi == 0.0) {
        stop = true;
      } else if (!std::isfinite(prev_hi)) {
        stop = false;
      } else {
        const double dmax = std::max(std::abs(prev_hi - in_lo), std::abs(in_hi - prev_lo));
        const double dmin = (prev_lo > in_hi) ? prev_lo - in_hi : (in_lo > prev_hi ? in_lo - prev_hi : 0.0);
        if (dmax < 1e-6 * in_lo) stop = true;
        else if (dmin >= 1e-6 * in_hi && in_lo > 0.0) stop = false;
        else certain = false, stop = false;
      }
      if (!certain) {  // exact sequential sums of this and the previous sweep
        double pe = 0.0;
        inertia_kernel<<<1, 1024, 0, st>>>(best.get(), n, inertia.get());
        launched(ctx);
        inertia.download(&in, 1, st);
        inertia_kernel<<<1, 1024, 0, st>>>(best_prev.get(), n, inertia.get());
        launched(ctx);
        inertia.download(&pe, 1, st);
        STGP_CUDA(cudaStreamSynchronize(st));
        stop = in == 0.0 || std::abs(pe - in) < 1e-6 * std::max(in, 1e-300);
      }
      if (stop) break;
      prev_lo = in_lo;
      prev_hi = in_hi;
      std::swap(best, best_prev);
      continue;
    }
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
    const int distinct = count_distinct_rows_device(ds->ctx, S.data(), n, 3);
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

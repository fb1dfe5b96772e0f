// Residual-correlation (d_r) neighbour search (neighbors.cpp:51-83, 324-329), bit-exact.
//
// d_r(i, j) = sqrt(max(1 - |k(p_i,p_j) - w_i.w_j| / sqrt(r_i r_j), 0)), w_i = L^{-1} k_m(p_i),
// r_i = sigma1_2 - |w_i|^2, degenerate (r <= 1e-7 sigma1_2) -> 1.  The selection
// kernel has no lag table (estimation.cpp:200,225).  Every reduction feeding d_r
// follows the oracle's order (sequential fused multiply-add chains in increasing
// index), so distances -- and hence index sets -- are bit-identical:
//   * Sigma_m Cholesky: left-looking, one column per step (single CTA);
//   * W: forward substitution as a column wavefront (each accumulator receives
//     its terms in increasing column order, the same sequence as the oracle);
//   * w_i.w_j: register-tiled Gram whose K loop runs sequentially per element.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>

#include "comm.hpp"
#include "lowrank_common.cuh"
#include "search.cuh"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

namespace {

// Sigma_m (live factors) + diagonal jitter, row-major M x M
__global__ void sel_sigma_kernel(const double* zx, const double* zy, const int32_t* ztid, int M, DevKernel k,
                                 LagTable lt, double jit1, double jit2, double* A) {
  const long long total = static_cast<long long>(M) * M;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / M), c = static_cast<int>(e % M);
    const int a = r >= c ? r : c, b = r >= c ? c : r;
    double pe, pb;
    lt.get2(ztid[a], ztid[b], pe, pb);
    TF f;
    f.pow_mE = pe;
    f.pow_mbh = pb;
    double v = gneiting_eval(k, spatial_dist(zx[a], zy[a], zx[b], zy[b]), f);
    if (r == c) {
      v = __dadd_rn(v, jit1);
      if (jit2 != 0.0) v = __dadd_rn(v, jit2);
    }
    A[e] = v;
  }
}

// Left-looking Cholesky in the oracle's order (chol_seq); A row-major in, L row-major out.
__global__ void __launch_bounds__(1024) chol_seq_kernel(const double* A, int M, double* L, int* fail) {
  __shared__ double diag;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int j = 0; j < M; ++j) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const double* Lj = L + static_cast<size_t>(j) * M;
      double acc = A[static_cast<size_t>(j) * M + j];
      for (int k = 0; k < j; ++k) acc = __fma_rn(-Lj[k], Lj[k], acc);
      if (acc <= 0.0) bad = 1;
      diag = __dsqrt_rn(acc);
      L[static_cast<size_t>(j) * M + j] = diag;
    }
    __syncthreads();
    if (bad) break;
    const double d = diag;
    const double* Lj = L + static_cast<size_t>(j) * M;
    for (int r = j + 1 + threadIdx.x; r < M; r += blockDim.x) {
      const double* Lr = L + static_cast<size_t>(r) * M;
      double s = A[static_cast<size_t>(r) * M + j];
      for (int k = 0; k < j; ++k) s = __fma_rn(-Lr[k], Lj[k], s);
      L[static_cast<size_t>(r) * M + j] = __ddiv_rn(s, d);
    }
  }
  if (threadIdx.x == 0 && bad) *fail = 1;
}

constexpr int kWB = 64;      // rows per block and columns per CTA
constexpr int kWKC = 16;     // K chunk of the off-diagonal update
constexpr int kWthreads = 256;
constexpr size_t kWsmem = sizeof(double) * (64 * 17 + 16 * 65 + 64 * 65 + 2 * 64 + 2 * 64) + sizeof(int) * 64;

// W(:, i) = L^{-1} k_m(p_i) for 64 columns per CTA.  Row blocks of 64: the
// off-diagonal part is a register-tiled update whose K loop runs in increasing
// c, the diagonal block is a column wavefront, so every accumulator receives
// -L[r][c] w_c for c = 0, 1, ... in order -- the oracle's fwd_seq sequence.
__global__ void __launch_bounds__(kWthreads) whiten_seq_kernel(const double* zx, const double* zy, const int32_t* ztid,
                                                              int M, int ldm, const double* x, const double* y,
                                                              const int32_t* tid, int n, DevKernel k, LagTable lt,
                                                              const double* L, double* W) {
  extern __shared__ double sm[];
  double* sL = sm;               // [64][17]
  double* sWt = sL + 64 * 17;    // [16][65]
  double* sD = sWt + 16 * 65;    // [64][65]
  double* wrow = sD + 64 * 65;   // [2][64]
  double* sx = wrow + 2 * 64;    // [64]
  double* sy = sx + 64;          // [64]
  int* st = reinterpret_cast<int*>(sy + 64);
  const int i0 = blockIdx.x * kWB;
  const int nc = min(kWB, n - i0);
  const int t = threadIdx.x;
  if (t < kWB) {
    const int i = i0 + (t < nc ? t : 0);
    sx[t] = x[i];
    sy[t] = y[i];
    st[t] = tid[i];
  }
  const int tr = (t / 16) * 4, tc = (t % 16) * 4;
  __syncthreads();
  for (int r0 = 0; r0 < M; r0 += kWB) {
    const int rb = min(kWB, M - r0);
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = r0 + tr + u, c = tc + v;
        double val = 0.0;
        if (r < M && c < nc) {
          double pe, pb;
          lt.get2(ztid[r], st[c], pe, pb);
          TF f;
          f.pow_mE = pe;
          f.pow_mbh = pb;
          val = gneiting_eval(k, spatial_dist(zx[r], zy[r], sx[c], sy[c]), f);  // k(z_r, p_i)
        }
        acc[u][v] = val;
      }
    for (int c0 = 0; c0 < r0; c0 += kWKC) {
      __syncthreads();
      for (int e = t; e < 64 * kWKC; e += kWthreads) {
        const int rr = e / kWKC, kk = e % kWKC;
        sL[rr * 17 + kk] = r0 + rr < M ? L[static_cast<size_t>(r0 + rr) * M + c0 + kk] : 0.0;
        const int cc = e / kWKC;
        sWt[kk * 65 + cc] = cc < nc ? W[static_cast<size_t>(i0 + cc) * ldm + c0 + kk] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kWKC; ++kk) {
        double lr[4], wv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) lr[u] = -sL[(tr + u) * 17 + kk];
#pragma unroll
        for (int v = 0; v < 4; ++v) wv[v] = sWt[kk * 65 + tc + v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = __fma_rn(lr[u], wv[v], acc[u][v]);
      }
    }
    __syncthreads();
    for (int e = t; e < 64 * 64; e += kWthreads) {
      const int rr = e / 64, cc = e % 64;
      sD[rr * 65 + cc] = (rr < rb && cc <= rr) ? L[static_cast<size_t>(r0 + rr) * M + r0 + cc] : 0.0;
    }
    __syncthreads();
    for (int cl = 0; cl < rb; ++cl) {
      double* buf = wrow + (cl & 1) * 64;
      if (cl >= tr && cl < tr + 4) {
        const double d = sD[cl * 65 + cl];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u == cl - tr)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const double wv = __ddiv_rn(acc[u][v], d);
              buf[tc + v] = wv;
              if (tc + v < nc) W[static_cast<size_t>(i0 + tc + v) * ldm + r0 + cl] = wv;
            }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = tr + u;
        if (rr > cl && rr < rb) {
          const double l = -sD[rr * 65 + cl];
#pragma unroll
          for (int v = 0; v < 4; ++v) acc[u][v] = __fma_rn(l, buf[tc + v], acc[u][v]);
        }
      }
    }
    __syncthreads();
  }
}

// r_i = sigma1_2 - |w_i|^2 (sequential fma from 0); degenerate flag
__global__ void resid_kernel(const double* W, int M, int ldm, int n, double s1, double* resid, int* degen) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* w = W + static_cast<size_t>(i) * ldm;
    double acc = 0.0;
    for (int k2 = 0; k2 < M; ++k2) acc = __fma_rn(w[k2], w[k2], acc);
    const double r = M > 0 ? __dsub_rn(s1, acc) : s1;
    resid[i] = r;
    degen[i] = r <= 1e-7 * s1 ? 1 : 0;
  }
}

// Per 64-row tile: time-id range, max |w| and min r over non-degenerate rows, degenerate flag.
__global__ void tile_stats_kernel(const double* resid, const int32_t* degen, const int32_t* tid, int n, double s1,
                                  int* tmin, int* tmax, double* wmax, double* rmin, int* hasdeg) {
  const int tile = blockIdx.x;
  const int i0 = tile * 64, i1 = min(n, i0 + 64);
  __shared__ double sw[64], sr[64];
  __shared__ int smn[64], smx[64], sdg[64];
  const int t = threadIdx.x;
  const int i = i0 + t;
  double w = 0.0, r = __longlong_as_double(0x7ff0000000000000LL);
  int mn = INT_MAX, mx = -1, dg = 0;
  if (i < i1) {
    mn = mx = tid[i];
    if (degen[i]) {
      dg = 1;
    } else {
      r = resid[i];
      w = s1 - resid[i];
    }
  }
  sw[t] = w;
  sr[t] = r;
  smn[t] = mn;
  smx[t] = mx;
  sdg[t] = dg;
  __syncthreads();
  for (int o = 32; o > 0; o >>= 1) {
    if (t < o) {
      sw[t] = fmax(sw[t], sw[t + o]);
      sr[t] = fmin(sr[t], sr[t + o]);
      smn[t] = min(smn[t], smn[t + o]);
      smx[t] = max(smx[t], smx[t + o]);
      sdg[t] = sdg[t] | sdg[t + o];
    }
    __syncthreads();
  }
  if (t == 0) {
    // |w|^2 = s1 - r up to one rounding of s1 (bounded by the 1e-11 factor of the prune test)
    wmax[tile] = sqrt(fmax(sw[0], 0.0) + 1e-15 * s1);
    rmin[tile] = sr[0];
    tmin[tile] = smn[0];
    tmax[tile] = smx[0];
    hasdeg[tile] = sdg[0];
  }
}

constexpr int kQT = 64;   // queries per CTA
constexpr int kCT = 64;   // candidates per tile
constexpr int kKC = 16;   // K chunk staged per pipeline stage
constexpr int kKS = kKC + 4;  // smem row stride (doubles): conflict-free DMMA fragment loads
constexpr int kStages = 3;
constexpr int kDrThreads = 256;

struct DrArgs {
  int n, m_v, M, ldm;  // ldm: multiple of kKC, rows [M, ldm) of W are zero
  const double *x, *y, *W, *resid;
  const int32_t *tid, *degen;
  DevKernel k;
  LagTable lt;
  int32_t* out;
  double* dist;
  // exact tile pruning
  const int *tmin, *tmax, *hasdeg;
  const double *wmax, *rmin;
  double s1;
  unsigned long long* stats;  // optional: [0] candidate tiles evaluated, [1] tiles pruned
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// Tiled exact d_r top-m over predecessors.  CTA = 64 consecutive queries; for each 64-candidate
// tile the Gram W_Q^T W_C is formed on the FP64 tensor pipe: mma.m8n8k4.f64 evaluates each
// element as the sequential fma chain over k (verified bit-identical on sm_100a,
// scripts/exp/dmma_order.cu), so G equals the oracle's chain exactly.  W chunks of kKC rows are
// staged by cp.async in a kStages ring; warp w owns the 16 x 32 sub-tile (rows 16 (w/2), cols
// 32 (w%2)).  The epilogue forms d_r, the warps merge the tile into per-query top-m lists.
constexpr size_t kDrStageDoubles = 2 * kQT * kKS;
constexpr size_t kDrSmem =
    sizeof(double) * (kStages * kDrStageDoubles + kQT * 32) + sizeof(int) * kQT * 32;
static_assert(kStages * kDrStageDoubles >= kQT * (kCT + 1), "distance tile aliases the stages");

__global__ void __launch_bounds__(kDrThreads) knn_dr_kernel(DrArgs a) {
  extern __shared__ double sm[];
  // the staging ring and the distance tile are never live together
  double* ring = sm;
  double (*sd)[kCT + 1] = reinterpret_cast<double (*)[kCT + 1]>(sm);
  double (*topd)[32] = reinterpret_cast<double (*)[32]>(sm + kStages * kDrStageDoubles);
  int (*topj)[32] = reinterpret_cast<int (*)[32]>(sm + kStages * kDrStageDoubles + kQT * 32);
  const int q0 = blockIdx.x * kQT;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  const int wr = wid >> 1, wc = wid & 1;  // warp sub-tile: rows 16 wr.., cols 32 wc..
  for (int e = tid; e < kQT * 32; e += kDrThreads) {
    topd[e / 32][e % 32] = __longlong_as_double(0x7ff0000000000000LL);
    topj[e / 32][e % 32] = INT_MAX;
  }
  const int qmax = min(q0 + kQT, a.n);
  __shared__ double s_dmax[kDrThreads / 32];
  __shared__ int s_prune;
  const int qtile = q0 / kQT;
  const int nch = a.ldm / kKC;
  // staging: thread copies 16 B pieces; a tile column chunk is kKC doubles = kKC/2 pieces
  constexpr int kPieces = 2 * kQT * (kKC / 2);  // Q and C
  static_assert(kPieces % kDrThreads == 0, "staging split");
  // candidate tiles nearest-first: tight thresholds early, then exact pruning of far tiles
  for (int c0 = ((qmax - 2) / kCT) * kCT; c0 >= 0; c0 -= kCT) {
    {
      // current worst threshold over the tile's queries (inf while any list is short)
      double dm = 0.0;
      for (int qq = tid; qq < kQT; qq += kDrThreads) {
        const int i = q0 + qq;
        if (i >= a.n) continue;
        const int m = min(a.m_v, i);
        if (m > 0) dm = fmax(dm, topd[qq][m - 1]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(kFull, dm, o));
      if (lane == 0) s_dmax[wid] = dm;
      __syncthreads();
      if (tid == 0) {
        double d = 0.0;
        for (int w2 = 0; w2 < kDrThreads / 32; ++w2) d = fmax(d, s_dmax[w2]);
        const int ct = c0 / kCT;
        int prune = 0;
        if (a.tmin && d < 1.0 && ct != qtile && !a.hasdeg[qtile]) {
          // rows are time sorted and C precedes Q, so the smallest lag is T(tmin_Q) - T(tmax_C).
          // |rho_r| <= |k| + |w_i||w_j| <= s1 T(u_min)^{-(delta+beta)} + wmax_Q wmax_C (non-degenerate
          // candidates; degenerate ones sit at d = 1 > d).  rmin_C = inf when all are degenerate.
          double pe, pb;
          a.lt.get2(a.tmin[qtile], a.tmax[ct], pe, pb);
          const double cmax =
              (a.s1 * pe + a.wmax[qtile] * a.wmax[ct]) * (1.0 + 1e-11) / sqrt(a.rmin[qtile] * a.rmin[ct]);
          if (cmax < 1.0 && (1.0 - cmax) - 1e-12 > d * d) prune = 1;
        }
        s_prune = prune;
        if (a.stats) atomicAdd(&a.stats[prune], 1ull);
      }
      __syncthreads();
      if (s_prune) continue;
    }
    double acc[2][4][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
    if (a.M > 0) {
      auto stage = [&](int ch) {
        double* sQ = ring + static_cast<size_t>(ch % kStages) * kDrStageDoubles;
        double* sC = sQ + kQT * kKS;
#pragma unroll
        for (int it = 0; it < kPieces / kDrThreads; ++it) {
          const int pc = tid + it * kDrThreads;
          const int which = pc / (kQT * (kKC / 2));  // 0: Q, 1: C
          const int rem = pc % (kQT * (kKC / 2));
          const int col = rem / (kKC / 2), piece = rem % (kKC / 2);
          const int g = min((which ? c0 : q0) + col, a.n - 1);
          cp_async16((which ? sC : sQ) + col * kKS + 2 * piece,
                     a.W + static_cast<size_t>(g) * a.ldm + static_cast<size_t>(ch) * kKC + 2 * piece);
        }
      };
#pragma unroll
      for (int ch = 0; ch < kStages - 1; ++ch) {
        if (ch < nch) stage(ch);
        cp_async_commit();
      }
      for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait<kStages - 2>();
        __syncthreads();  // chunk ch visible; the stage about to be refilled is no longer read
        if (ch + kStages - 1 < nch) stage(ch + kStages - 1);
        cp_async_commit();
        const double* sQ = ring + static_cast<size_t>(ch % kStages) * kDrStageDoubles;
        const double* sC = sQ + kQT * kKS;
#pragma unroll
        for (int kb = 0; kb < kKC; kb += 4) {
          double fa[2], fb[4];
#pragma unroll
          for (int u = 0; u < 2; ++u) fa[u] = sQ[(16 * wr + 8 * u + grp) * kKS + kb + tig];
#pragma unroll
          for (int v = 0; v < 4; ++v) fb[v] = sC[(32 * wc + 8 * v + grp) * kKS + kb + tig];
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) dmma_f64(acc[u][v][0], acc[u][v][1], fa[u], fb[v]);
        }
      }
      cp_async_wait<0>();
    }
    // epilogue: d_r for the thread's 16 pairs (sd aliases the staging ring)
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int qq = 16 * wr + 8 * u + grp, cc = 32 * wc + 8 * v + 2 * tig + h;
          const int i = q0 + qq, j = c0 + cc;
          double d = __longlong_as_double(0x7ff0000000000000LL);
          if (i < a.n && j < i) {
            if (a.degen[i] || a.degen[j]) {
              d = 1.0;
            } else {
              double pe, pb;
              a.lt.get2(a.tid[i], a.tid[j], pe, pb);
              TF f;
              f.pow_mE = pe;
              f.pow_mbh = pb;
              double rho = gneiting_eval(a.k, spatial_dist(a.x[i], a.y[i], a.x[j], a.y[j]), f);
              if (a.M > 0) rho = __dsub_rn(rho, acc[u][v][h]);
              const double rad =
                  __dsub_rn(1.0, __ddiv_rn(fabs(rho), __dsqrt_rn(__dmul_rn(a.resid[i], a.resid[j]))));
              d = __dsqrt_rn(rad < 0.0 ? 0.0 : rad);
            }
          }
          sd[qq][cc] = d;
        }
    __syncthreads();
    // merge: warp wid handles queries wid, wid + 8, ...
    for (int qq = wid; qq < kQT; qq += kDrThreads / 32) {
      const int i = q0 + qq;
      if (i >= a.n) break;
      const int m = min(a.m_v, i);
      if (m <= 0) continue;
      TopM e{topd[qq][lane], topj[qq][lane]};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = lane + 32 * h;
        const int j = c0 + cc;
        const double d = sd[qq][cc];
        const double wd = __shfl_sync(kFull, e.d, m - 1);
        const int wj = __shfl_sync(kFull, e.j, m - 1);
        const unsigned acc = __ballot_sync(kFull, j < i && lex_less(d, j, wd, wj));
        if (acc) topm_insert(e, m, acc, d, j, lane);
      }
      topd[qq][lane] = e.d;
      topj[qq][lane] = e.j;
    }
  }
  __syncthreads();
  for (int qq = wid; qq < kQT; qq += kDrThreads / 32) {
    const int i = q0 + qq;
    if (i >= a.n) break;
    const int m = min(a.m_v, i);
    TopM e{topd[qq][lane], topj[qq][lane]};
    topm_emit(e, a.m_v, m, lane, a.out + static_cast<size_t>(i) * a.m_v, a.dist ? a.dist + static_cast<size_t>(i) * a.m_v : nullptr);
  }
}

}  // namespace

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

int stgp_residual_neighbors(stgp_dataset* ds, const stgp_params* theta, const stgp_inducing* ind, int m_v,
                            stgp_neighbors** out) {
  return guarded([&] {
    if (!ds || !theta || !ind || !out) config_error("stgp_residual_neighbors: null argument");
    if (m_v < 0) config_error("m_v must be >= 0");
    if (m_v > 32) config_error("neighbour search supports m_v <= 32 on the device");
    Params p;
    std::memcpy(&p, theta, sizeof(p));
    validate_params(p);
    stgp_ctx* ctx = ds->ctx;
    cudaStream_t st = ctx->stream;
    const int n = ds->n, M = ind->M();
    const DevKernel k = dev_kernel(p);
    // time index over data + inducing times, live factors (no lag table in the selection kernel)
    std::vector<double> zx(M), zy(M), zt(M);
    for (int j = 0; j < M; ++j) {
      zx[j] = ind->xyt[3 * j];
      zy[j] = ind->xyt[3 * j + 1];
      zt[j] = ind->xyt[3 * j + 2];
    }
    std::set<double> it(zt.begin(), zt.end());
    std::vector<double> Ti(it.begin(), it.end());
    TimeIndex ti;
    ti.T = ds->Tdata;
    ti.T.insert(ti.T.end(), Ti.begin(), Ti.end());
    ti.build();
    DevLagTable dl;
    LagPolicy live;
    upload_lag_table(dl, ti, p, live, st, true);
    const LagTable lt = lag_view(dl);
    std::vector<int32_t> ztid(M);
    const int nD = static_cast<int>(ds->Tdata.size());
    for (int j = 0; j < M; ++j)
      ztid[j] = nD + static_cast<int>(std::lower_bound(Ti.begin(), Ti.end(), zt[j]) - Ti.begin());
    DevBuf<double> dzx, dzy;
    DevBuf<int32_t> dzt;
    dzx.upload(zx.data(), M, st);
    dzy.upload(zy.data(), M, st);
    dzt.upload(ztid.data(), M, st);
    const int ldm = std::max(kKC, (M + kKC - 1) / kKC * kKC);  // zero rows [M, ldm): exact extra fma(0, 0, g)
    DevBuf<double> W(static_cast<size_t>(ldm) * n), resid(n);
    STGP_CUDA(cudaMemsetAsync(W.get(), 0, sizeof(double) * ldm * n, st));
    DevBuf<int32_t> degen(n);
    {
      ProfRegion pr(ctx, "dr_whiten");
      if (M > 0) {
        // InducingBasis(set, selection kernel): jittered Sigma_m, one retry at 10x (inducing.cpp:250-261)
        DevBuf<double> A(static_cast<size_t>(M) * M), L(static_cast<size_t>(M) * M);
        DevBuf<int> fail(1);
        const double jitter = 1e-8 * p.sigma1_2;
        bool ok = false;
        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
          sel_sigma_kernel<<<grid_for(static_cast<long long>(M) * M), 256, 0, st>>>(
              dzx.get(), dzy.get(), dzt.get(), M, k, lt, jitter, attempt == 0 ? 0.0 : 9.0 * jitter, A.get());
          launched(ctx);
          fail.zero(st);
          chol_seq_kernel<<<1, 1024, 0, st>>>(A.get(), M, L.get(), fail.get());
          launched(ctx);
          int f = 0;
          fail.download(&f, 1, st);
          STGP_CUDA(cudaStreamSynchronize(st));
          ok = f == 0;
        }
        if (!ok) numeric_error("InducingBasis: inducing covariance is not positive definite");
        STGP_CUDA(cudaFuncSetAttribute(whiten_seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kWsmem)));
        whiten_seq_kernel<<<ceil_div(n, kWB), kWthreads, kWsmem, st>>>(dzx.get(), dzy.get(), dzt.get(), M, ldm,
                                                                      ds->x.get(), ds->y.get(), ds->tid.get(), n, k, lt,
                                                                      L.get(), W.get());
        launched(ctx);
      }
      resid_kernel<<<grid_for(n), 256, 0, st>>>(W.get(), M, ldm, n, p.sigma1_2, resid.get(), degen.get());
      launched(ctx);
    }
    auto nb = std::make_unique<stgp_neighbors>();
    nb->ctx = ctx;
    nb->n = n;
    nb->m_v = std::max(m_v, 1);
    nb->kind = STGP_METRIC_DR;
    const size_t total = static_cast<size_t>(n) * nb->m_v;
    nb->idx.alloc(total);
    nb->dist.alloc(total);
    nb->has_dist = true;
    if (m_v == 0) {
      std::vector<int32_t> neg(total, -1);
      nb->idx.upload(neg.data(), total, st);
    } else {
      DrArgs a{};
      a.n = n;
      a.m_v = m_v;
      a.M = M;
      a.ldm = ldm;
      a.x = ds->x.get();
      a.y = ds->y.get();
      a.W = W.get();
      a.resid = resid.get();
      a.tid = ds->tid.get();
      a.degen = degen.get();
      a.k = k;
      a.lt = lt;
      a.out = nb->idx.get();
      a.dist = nb->dist.get();
      const int ntile = ceil_div(n, 64);
      DevBuf<int> tmn(ntile), tmx(ntile), hdg(ntile);
      DevBuf<double> wmx(ntile), rmn(ntile);
      tile_stats_kernel<<<ntile, 64, 0, st>>>(resid.get(), degen.get(), ds->tid.get(), n, p.sigma1_2, tmn.get(),
                                              tmx.get(), wmx.get(), rmn.get(), hdg.get());
      launched(ctx);
      a.tmin = tmn.get();
      a.tmax = tmx.get();
      a.wmax = wmx.get();
      a.rmin = rmn.get();
      a.hasdeg = hdg.get();
      a.s1 = p.sigma1_2;
      // pruning needs time-sorted rows (tile time ranges); otherwise plain brute force
      if (!ds->time_sorted) a.tmin = nullptr;
      DevBuf<unsigned long long> stats;
      if (std::getenv("STGP_DR_STATS")) {  // diagnostics: tile pairs evaluated / pruned
        stats.alloc(2);
        STGP_CUDA(cudaMemsetAsync(stats.get(), 0, 16, st));
        a.stats = stats.get();
      }
      ProfRegion pr(ctx, "knn_dr");
      STGP_CUDA(cudaFuncSetAttribute(knn_dr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(kDrSmem)));
      knn_dr_kernel<<<ceil_div(n, kQT), kDrThreads, kDrSmem, st>>>(a);
      launched(ctx);
      if (a.stats) {
        unsigned long long h[2];
        STGP_CUDA(cudaMemcpyAsync(h, a.stats, 16, cudaMemcpyDeviceToHost, st));
        STGP_CUDA(cudaStreamSynchronize(st));
        std::fprintf(stderr, "[stgp] d_r tiles: evaluated %llu pruned %llu\n", h[0], h[1]);
      }
    }
    STGP_CUDA(cudaStreamSynchronize(st));
    prof_collect(ctx);
    *out = nb.release();
  });
}

}  // extern "C"

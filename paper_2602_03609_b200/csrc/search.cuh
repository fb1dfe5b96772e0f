// Exact predecessor kNN kernels (K8 of SURVEY.md §2.4).
//
// Semantics: for query i the m = min(m_v, i) predecessors j < i with the
// smallest (d(i, j), j) in lexicographic order, returned ascending by index --
// the reference's brute_force_knn (tests/oracles.cpp:157-168), which its cover
// tree provably equals (test_neighbors.cpp:96-131), and euclidean_neighbors
// (neighbors.cpp:257-316).  d values are bit-identical to the host metric
// (gneiting.cuh), so the index sets are bit-exact.
//
// One warp per query; the running top-m list is spread over the lanes (lane l
// holds the l-th best (d, j)), candidates are evaluated 32 at a time and
// inserted with a ballot + shfl_up.  Data rows are time ordered, so equal-time
// blocks are scanned backwards from the query's own block; a whole block is
// skipped when the exact lag bound proves every candidate in it is worse than
// the current m-th best (d_c: |rho| <= T(u)^{-(delta+beta)} because the Matern
// factor is <= 1; euclid: d^2 >= dt^2).
#pragma once

#include <climits>

#include "common.cuh"
#include "gneiting.cuh"
#include "rows.cuh"

namespace stgp {

struct SearchArgs {
  int n, m_v;
  int q_begin, q_end;
  const double *x, *y, *t;
  const int32_t* tid;
  const int32_t* blk_of;     // data block of each row (time-sorted data), or null
  const int32_t* blk_start;  // nblk + 1
  const int32_t* blk_tid;    // tid of each block
  int nblk;
  DevKernel k;
  LagTable lt;  // live temporal factors (selection kernel, no lag table)
  double ss, ts;  // euclid scales
  int32_t* out;   // (q_end - q_begin) * m_v
  double* dist;   // optional, sorted by distance
};

struct TopM {
  double d;
  int j;
};

__device__ __forceinline__ bool lex_less(double d1, int j1, double d2, int j2) {
  return d1 < d2 || (d1 == d2 && j1 < j2);
}

// Insert the candidates held by lanes in `mask` (each lane's (cd, cj)).
__device__ __forceinline__ void topm_insert(TopM& e, int m, unsigned mask, double cd, int cj, int lane) {
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const double d = __shfl_sync(kFull, cd, src);
    const int j = __shfl_sync(kFull, cj, src);
    const double wd = __shfl_sync(kFull, e.d, m - 1);
    const int wj = __shfl_sync(kFull, e.j, m - 1);
    if (!lex_less(d, j, wd, wj)) continue;
    const bool less = lane < m && lex_less(e.d, e.j, d, j);
    const int pos = __popc(__ballot_sync(kFull, less));
    const double ud = __shfl_up_sync(kFull, e.d, 1);
    const int uj = __shfl_up_sync(kFull, e.j, 1);
    if (lane < m) {
      if (lane == pos) {
        e.d = d;
        e.j = j;
      } else if (lane > pos) {
        e.d = ud;
        e.j = uj;
      }
    }
  }
}

// Write the list ascending by index; distances (optional) ascending by (d, j).
__device__ __forceinline__ void topm_emit(const TopM& e, int m_v, int m, int lane, int32_t* orow, double* drow) {
  const bool valid = lane < m && e.j != INT_MAX;
  int rank = 0;
  for (int s = 0; s < 32; ++s) {
    const int oj = __shfl_sync(kFull, e.j, s);
    const bool ov = __shfl_sync(kFull, valid ? 1 : 0, s) != 0;
    if (ov && oj < e.j) ++rank;
  }
  if (lane < m_v) {
    orow[lane] = -1;
    if (drow) drow[lane] = __longlong_as_double(0x7ff8000000000000LL);
  }
  __syncwarp();
  if (valid) {
    STGP_DCHECK(rank < m);
    orow[rank] = e.j;
    if (drow) drow[lane] = e.d;
  }
}

// Lists longer than a warp (32 < m <= 32 R): slot s = 32 r + lane lives in e[r] of that lane, slots
// ascending by (d, j).  For R = 1 these reduce to topm_insert / topm_emit above.
template <int R>
__device__ __forceinline__ void topl_init(TopM (&e)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) e[r] = TopM{__longlong_as_double(0x7ff0000000000000LL), INT_MAX};
}

template <int R>
__device__ __forceinline__ void topl_worst(const TopM (&e)[R], int m, double& wd, int& wj) {
  const int rw = (m - 1) >> 5;
  double d = e[0].d;
  int j = e[0].j;
#pragma unroll
  for (int r = 1; r < R; ++r)
    if (r == rw) {
      d = e[r].d;
      j = e[r].j;
    }
  wd = __shfl_sync(kFull, d, (m - 1) & 31);
  wj = __shfl_sync(kFull, j, (m - 1) & 31);
}

template <int R>
__device__ __forceinline__ void topl_insert(TopM (&e)[R], int m, unsigned mask, double cd, int cj, int lane) {
  while (mask) {
    const int src = __ffs(mask) - 1;
    mask &= mask - 1;
    const double d = __shfl_sync(kFull, cd, src);
    const int j = __shfl_sync(kFull, cj, src);
    double wd;
    int wj;
    topl_worst(e, m, wd, wj);
    if (!lex_less(d, j, wd, wj)) continue;
    int pos = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) pos += __popc(__ballot_sync(kFull, 32 * r + lane < m && lex_less(e[r].d, e[r].j, d, j)));
    double ud[R];
    int uj[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ud[r] = __shfl_up_sync(kFull, e[r].d, 1);
      uj[r] = __shfl_up_sync(kFull, e[r].j, 1);
    }
#pragma unroll
    for (int r = 1; r < R; ++r) {  // slot 32 r takes slot 32 r - 1 (lane 31 of the row below)
      const double ld = __shfl_sync(kFull, e[r - 1].d, 31);
      const int lj = __shfl_sync(kFull, e[r - 1].j, 31);
      if (lane == 0) {
        ud[r] = ld;
        uj[r] = lj;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int slot = 32 * r + lane;
      if (slot < m) {
        if (slot == pos) {
          e[r].d = d;
          e[r].j = j;
        } else if (slot > pos) {
          e[r].d = ud[r];
          e[r].j = uj[r];
        }
      }
    }
  }
}

// Write the list ascending by index; distances (optional) ascending by (d, j).
template <int R>
__device__ __forceinline__ void topl_emit(const TopM (&e)[R], int m_v, int m, int lane, int32_t* orow, double* drow) {
  bool valid[R];
  int rank[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    valid[r] = 32 * r + lane < m && e[r].j != INT_MAX;
    rank[r] = 0;
  }
#pragma unroll
  for (int rr = 0; rr < R; ++rr)
    for (int s = 0; s < 32; ++s) {
      const int oj = __shfl_sync(kFull, e[rr].j, s);
      const bool ov = __shfl_sync(kFull, valid[rr] ? 1 : 0, s) != 0;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (ov && oj < e[r].j) ++rank[r];
    }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int slot = 32 * r + lane;
    if (slot < m_v) {
      orow[slot] = -1;
      if (drow) drow[slot] = __longlong_as_double(0x7ff8000000000000LL);
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (valid[r]) {
      STGP_DCHECK(rank[r] < m);
      orow[rank[r]] = e[r].j;
      if (drow) drow[32 * r + lane] = e[r].d;
    }
}

// d_c(i, j) = sqrt(max(1 - |k(p_i, p_j) / sigma1_2|, 0))   (neighbors.cpp:37-43)
template <bool GEN>
__device__ __forceinline__ double dc_value(const DevKernel& k, double xi, double yi, double xj, double yj,
                                           double pow_mE, double pow_mbh) {
  TF f;
  f.pow_mE = pow_mE;
  f.pow_mbh = pow_mbh;
  const double cov = gneiting_eval<GEN>(k, spatial_dist(xi, yi, xj, yj), f);
  const double rho = __ddiv_rn(cov, k.s1);
  const double rad = __dsub_rn(1.0, fabs(rho));
  return __dsqrt_rn(rad < 0.0 ? 0.0 : rad);
}

// METRIC 0: d_c, 1: euclid (squared scaled distance); GEN: general nu; R: list slots per lane (m_v <= 32 R)
template <int METRIC, bool GEN = false, int R = 1>
__global__ void __launch_bounds__(256) knn_kernel(SearchArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int i = a.q_begin + gw; i < a.q_end; i += nw) {
    const int m = a.m_v < i ? a.m_v : i;
    TopM e[R];
    topl_init(e);
    const double xi = a.x[i], yi = a.y[i];
    double sxi = 0, syi = 0, sti = 0;
    if (METRIC == 1) {
      sxi = __ddiv_rn(xi, a.ss);
      syi = __ddiv_rn(yi, a.ss);
      sti = __ddiv_rn(a.t[i], a.ts);
    }
    const int ti = a.tid[i];
    const int bi = a.blk_of ? a.blk_of[i] : 0;
    const int nb_scan = a.blk_of ? bi + 1 : 1;
    for (int bb = 0; bb < nb_scan && m > 0; ++bb) {
      int s, eend;
      double pe = 0, pbh = 0, dt2 = 0;
      if (a.blk_of) {
        const int b = bi - bb;
        s = a.blk_start[b];
        eend = min(a.blk_start[b + 1], i);
        if (METRIC == 0) {
          a.lt.get2(ti, a.blk_tid[b], pe, pbh);
          double wd;
          int wj;
          topl_worst(e, m, wd, wj);
          // exact prune: every d^2 in the block >= 1 - T^{-(delta+beta)} - O(eps)
          if (wd != __longlong_as_double(0x7ff0000000000000LL) && (1.0 - pe) - 1e-12 > wd * wd) continue;
        } else {
          const double dt = __dsub_rn(sti, __ddiv_rn(a.t[s], a.ts));
          dt2 = __dmul_rn(dt, dt);
          double wd;
          int wj;
          topl_worst(e, m, wd, wj);
          if (dt2 > wd) continue;
        }
      } else {
        s = 0;
        eend = i;
      }
      for (int j0 = s; j0 < eend; j0 += 32) {
        const int j = j0 + lane;
        double d = __longlong_as_double(0x7ff0000000000000LL);
        if (j < eend) {
          const double xj = __ldg(&a.x[j]), yj = __ldg(&a.y[j]);
          if (METRIC == 0) {
            if (!a.blk_of) a.lt.get2(ti, __ldg(&a.tid[j]), pe, pbh);
            d = dc_value<GEN>(a.k, xi, yi, xj, yj, pe, pbh);
          } else {
            const double dx = __dsub_rn(sxi, __ddiv_rn(xj, a.ss));
            const double dy = __dsub_rn(syi, __ddiv_rn(yj, a.ss));
            d = __dadd_rn(__dadd_rn(dt2, __dmul_rn(dx, dx)), __dmul_rn(dy, dy));
          }
        }
        double wd;
        int wj;
        topl_worst(e, m, wd, wj);
        const unsigned acc = __ballot_sync(kFull, j < eend && lex_less(d, j, wd, wj));
        if (acc) topl_insert(e, m, acc, d, j, lane);
      }
    }
    const size_t o = static_cast<size_t>(i - a.q_begin) * a.m_v;
    topl_emit(e, a.m_v, m, lane, a.out + o, a.dist ? a.dist + o : nullptr);
  }
}

}  // namespace stgp

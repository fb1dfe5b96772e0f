// Prediction (approximations.cpp:806-1080) and GLS coefficients (approximations.cpp:752-798).
//
// Target neighbour sets (target_neighbors, approximations.cpp:816-863) are exact
// top-m over ALL training rows under the structure's metric with un-rooted
// distances; equal-time blocks are visited nearest-in-time first and skipped by
// the same exact lag bounds as the searches.  The per-target conditional solves
// are small (k <= pred_m_v) and run one thread per target.
//
// VIF predictive variance, whitened (wq = L_m^{-1} u_p, sN = A on N):
//   var = |wq|^2 + D_p - 2 wq.(W sN) - wq'(K - I) wq + h' K^{-1} h,  h = W sN + (K - I) wq,
// which is the reference's var_prior - quad (approximations.cpp:1050-1072) with the two
// O(n) sparse triangular solves per target cancelled algebraically:
// sN' Sigma_s sN appears in both var_prior and cp'qc.
#include <algorithm>
#include <climits>
#include <cstring>
#include <memory>
#include <set>

#include "comm.hpp"
#include "dense.cuh"
#include "lowrank_common.cuh"
#include "rows.cuh"
#include "search.cuh"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

namespace {


struct PredArgs {
  int n, np, m;  // training rows, targets, pred_m_v
  const double *x, *y, *t;
  const int32_t* tid;
  const double *qx, *qy, *qt;
  const int32_t* qtid;
  int metric;  // 0 euclid, 1 d_c, 2 d_r
  double ss, ts;
  DevKernel k;
  LagTable lt;
  double s1;
  // time-sorted blocks of the training data
  const int32_t* blk_start;
  const double* Tdata;
  int nblk;
  // d_r: whitened columns, residual variances
  const double* W;
  int ldm, M;
  const double* resid;
  const double* Wq;     // ldm x np
  const double* rq;     // np
  // d_r pruning: |w_j|^2 (n), |w_q|^2 (np); per time block min r and max |w| / sqrt(r) over its
  // non-degenerate rows
  const double *wsq, *wqsq, *blk_rmin, *blk_amax;
  int32_t* nbr_out;     // np x m (ascending)
  double* scratch_d;    // np x n (generic path)
};

// wd: the target's current worst list entry (inf while short).  d_r returns +inf for a candidate
// that provably cannot beat it: |k - w_q.w_j| <= |k| + |w_q||w_j| (skips the M-long dot product).
__device__ __forceinline__ double target_dist(const PredArgs& a, int p, int j, double wd) {
  if (a.metric == 0) {
    const double dx = __ddiv_rn(__dsub_rn(a.qx[p], a.x[j]), a.ss);
    const double dy = __ddiv_rn(__dsub_rn(a.qy[p], a.y[j]), a.ss);
    const double dt = __ddiv_rn(__dsub_rn(a.qt[p], a.t[j]), a.ts);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dt, dt));
  }
  double pe, pb;
  a.lt.get2(a.qtid[p], a.tid[j], pe, pb);
  TF f;
  f.pow_mE = pe;
  f.pow_mbh = pb;
  const double cov = gneiting_eval<true>(a.k, spatial_dist(a.qx[p], a.qy[p], a.x[j], a.y[j]), f);  // kernel(q, p_j)
  if (a.metric == 1) return __dsub_rn(1.0, fabs(__ddiv_rn(cov, a.s1)));
  const double tol = 1e-7 * a.s1;
  const double dj = a.resid[j], rq = a.rq[p];
  if (dj <= tol || rq <= tol) return 1.0;
  double rho = cov;
  if (a.M > 0 && a.wsq && wd < 1.0) {
    const double ub = (fabs(cov) + sqrt(a.wqsq[p] * a.wsq[j]) * (1.0 + 1e-12)) / sqrt(dj * rq) * (1.0 + 1e-11);
    if ((1.0 - ub) - 1e-12 > wd) return __longlong_as_double(0x7ff0000000000000LL);
  }
  if (a.M > 0) {
    const double* wq = a.Wq + static_cast<size_t>(p) * a.ldm;
    const double* wj = a.W + static_cast<size_t>(j) * a.ldm;
    double s = 0.0;
    for (int k2 = 0; k2 < a.M; ++k2) s = __fma_rn(wq[k2], wj[k2], s);
    rho = __dsub_rn(rho, s);
  }
  return __dsub_rn(1.0, __ddiv_rn(fabs(rho), __dsqrt_rn(__dmul_rn(dj, rq))));
}

// per time block: min r and max |w| / sqrt(r) over its non-degenerate rows (inf / 0 when none)
__global__ void __launch_bounds__(256) block_bound_kernel(int nblk, const int32_t* blk_start, const double* resid,
                                                          const double* wsq, double s1, double* rmin, double* amax) {
  __shared__ double sr[256], sa[256];
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    double r0 = __longlong_as_double(0x7ff0000000000000LL), a0 = 0.0;
    for (int j = blk_start[b] + threadIdx.x; j < blk_start[b + 1]; j += blockDim.x) {
      const double r = resid[j];
      if (r > 1e-7 * s1) {
        r0 = fmin(r0, r);
        a0 = fmax(a0, sqrt(wsq[j] / r) * (1.0 + 1e-12));
      }
    }
    sr[threadIdx.x] = r0;
    sa[threadIdx.x] = a0;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        sr[threadIdx.x] = fmin(sr[threadIdx.x], sr[threadIdx.x + o]);
        sa[threadIdx.x] = fmax(sa[threadIdx.x], sa[threadIdx.x + o]);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      rmin[b] = sr[0];
      amax[b] = sa[0];
    }
    __syncthreads();
  }
}

// warp per target, m <= 32: exact top-m over all rows, nearest time blocks first
__global__ void __launch_bounds__(256) target_knn_kernel(PredArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < a.np; p += nw) {
    const int m = min(a.m, a.n);
    TopM e{__longlong_as_double(0x7ff0000000000000LL), INT_MAX};
    const double tq = a.qt[p];
    // block position: first block with T_b >= t_q
    int lo = 0, hi = a.nblk;
    if (a.blk_start) {
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a.Tdata[mid] < tq) lo = mid + 1;
        else hi = mid;
      }
    }
    int L = lo - 1, R = lo;
    const int nsteps = a.blk_start ? a.nblk : 1;
    for (int step = 0; step < nsteps; ++step) {
      int s0, s1e;
      if (a.blk_start) {
        int b;
        if (L < 0) b = R++;
        else if (R >= a.nblk) b = L--;
        else if (tq - a.Tdata[L] <= a.Tdata[R] - tq) b = L--;
        else b = R++;
        s0 = a.blk_start[b];
        s1e = a.blk_start[b + 1];
        const double wd = __shfl_sync(kFull, e.d, m - 1);
        if (wd != __longlong_as_double(0x7ff0000000000000LL)) {
          if (a.metric == 0) {
            const double dt = __ddiv_rn(__dsub_rn(tq, a.Tdata[b]), a.ts);
            if (__dmul_rn(dt, dt) > wd) continue;
          } else if (a.metric == 1) {
            double pe, pb;
            a.lt.get2(a.qtid[p], a.tid[s0], pe, pb);
            if ((1.0 - pe) - 1e-12 > wd) continue;
          } else if (a.M > 0 && a.blk_amax && wd < 1.0 && a.rq[p] > 1e-7 * a.s1) {
            // d_r block bound: s1 T(u)^-E / sqrt(r_q rmin_b) + a_q amax_b (degenerate rows sit at d = 1)
            double pe, pb;
            a.lt.get2(a.qtid[p], a.tid[s0], pe, pb);
            const double rq = a.rq[p];
            const double cb = (a.s1 * pe / sqrt(rq * a.blk_rmin[b]) + sqrt(a.wqsq[p] / rq) * a.blk_amax[b]) *
                              (1.0 + 1e-11);
            if (cb < 1.0 && (1.0 - cb) - 1e-12 > wd) continue;
          }
        }
      } else {
        s0 = 0;
        s1e = a.n;
      }
      for (int j0 = s0; j0 < s1e; j0 += 32) {
        const int j = j0 + lane;
        double d = __longlong_as_double(0x7ff0000000000000LL);
        const double wd = __shfl_sync(kFull, e.d, m - 1);
        if (j < s1e) d = target_dist(a, p, j, wd);
        const int wj = __shfl_sync(kFull, e.j, m - 1);
        const unsigned acc = __ballot_sync(kFull, j < s1e && lex_less(d, j, wd, wj));
        if (acc) topm_insert(e, m, acc, d, j, lane);
      }
    }
    topm_emit(e, a.m, m, lane, a.nbr_out + static_cast<size_t>(p) * a.m, nullptr);
  }
}

// generic path (m > 32): thread per target, distances to all rows, selection by (d, j)
__global__ void target_knn_generic_kernel(PredArgs a) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < a.np; p += gridDim.x * blockDim.x) {
    double* d = a.scratch_d + static_cast<size_t>(p) * a.n;
    for (int j = 0; j < a.n; ++j) d[j] = target_dist(a, p, j, __longlong_as_double(0x7ff0000000000000LL));
    const int m = min(a.m, a.n);
    int32_t* out = a.nbr_out + static_cast<size_t>(p) * a.m;
    // m rounds of arg-min over the remaining rows (ties to the smaller index)
    for (int r = 0; r < m; ++r) {
      int best = -1;
      for (int j = 0; j < a.n; ++j)
        if (best < 0 || lex_less(d[j], j, d[best], best)) best = j;
      out[r] = best;
      d[best] = __longlong_as_double(0x7ff0000000000000LL);  // taken (distances are finite)
    }
    for (int r = m; r < a.m; ++r) out[r] = -1;
    // ascending
    for (int r = 1; r < m; ++r) {
      const int v = out[r];
      int q = r - 1;
      while (q >= 0 && out[q] > v) {
        out[q + 1] = out[q];
        --q;
      }
      out[q + 1] = v;
    }
  }
}

struct CondArgs {
  int np, m, n;
  const int32_t* nbr;  // np x m ascending, -1 padded
  const double *x, *y, *qx, *qy;
  const int32_t *tid, *qtid;
  DevKernel k;
  LagTable lt;
  double s1, sigma2;
  const double* r;  // residual (Vecchia) or z (VIF)
  // VIF residual covariances
  const double* W;
  int ldm, M;
  const double* Wq;
  const double* rq;
  double* mu_part;  // np
  double* var_out;  // np: Vecchia var; VIF D_p
  double* A_out;    // np x m (VIF: for W sN)
  double* scratch;  // per-thread k x k + 2k
  int* fail;
  int laplace;  // Laplace target rows (approximations.cpp:1135-1146, 1320-1331): no nugget, C + 1e-10 s1, no retry
};

// thread per target: conditional block over N with one jitter retry (approximations.cpp:889-913, 1016-1043)
__global__ void cond_solve_kernel(CondArgs a, bool vif) {
  const int K = a.m;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < a.np; p += gridDim.x * blockDim.x) {
    double* C = a.scratch + static_cast<size_t>(p) * (static_cast<size_t>(K) * K + 2 * K);
    double* c = C + static_cast<size_t>(K) * K;
    double* A = c + K;
    const int32_t* N = a.nbr + static_cast<size_t>(p) * K;
    int k = 0;
    while (k < K && N[k] >= 0) ++k;
    auto wdot = [&](const double* u, const double* v) {
      double s = 0.0;
      for (int q = 0; q < a.M; ++q) s = fma(u[q], v[q], s);
      return s;
    };
    const double* wq = vif ? a.Wq + static_cast<size_t>(p) * a.ldm : nullptr;
    for (int i = 0; i < k; ++i) {
      const int ja = N[i];
      double pe, pb;
      a.lt.get2(a.qtid[p], a.tid[ja], pe, pb);
      TF f;
      f.pow_mE = pe;
      f.pow_mbh = pb;
      double va = gneiting_eval<true>(a.k, spatial_dist(a.qx[p], a.qy[p], a.x[ja], a.y[ja]), f);
      if (vif && a.M > 0) va -= wdot(wq, a.W + static_cast<size_t>(ja) * a.ldm);
      c[i] = va;
      for (int b = 0; b <= i; ++b) {
        const int jb = N[b];
        a.lt.get2(a.tid[ja], a.tid[jb], pe, pb);
        f.pow_mE = pe;
        f.pow_mbh = pb;
        double v = gneiting_eval<true>(a.k, spatial_dist(a.x[ja], a.y[ja], a.x[jb], a.y[jb]), f);
        if (vif && a.M > 0) v -= wdot(a.W + static_cast<size_t>(ja) * a.ldm, a.W + static_cast<size_t>(jb) * a.ldm);
        if (i == b) v += a.sigma2;
        C[i * K + b] = v;
        C[b * K + i] = v;
      }
    }
    bool ok = false;
    for (int attempt = a.laplace ? 1 : 0; attempt < 2 && !ok; ++attempt) {
      // restore the lower triangle from the upper one (diagonal kept in A[] on the first pass)
      for (int i = 0; i < k; ++i) {
        if (attempt == 0 || a.laplace) A[i] = C[i * K + i];
        for (int b = 0; b < i; ++b) C[i * K + b] = C[b * K + i];
        C[i * K + i] = attempt == 0 ? A[i] : A[i] + 1e-10 * a.s1;
      }
      bool good = true;
      for (int j = 0; j < k && good; ++j) {
        double s = C[j * K + j];
        for (int q = 0; q < j; ++q) s = fma(-C[j * K + q], C[j * K + q], s);
        if (!(s > 0.0)) {
          good = false;
          break;
        }
        const double d = sqrt(s);
        C[j * K + j] = d;
        for (int r = j + 1; r < k; ++r) {
          double v = C[r * K + j];
          for (int q = 0; q < j; ++q) v = fma(-C[r * K + q], C[j * K + q], v);
          C[r * K + j] = v / d;
        }
      }
      ok = good;
    }
    if (!ok) {
      atomicExch(a.fail, 1);
      continue;
    }
    for (int r = 0; r < k; ++r) {
      double s = c[r];
      for (int q = 0; q < r; ++q) s = fma(-C[r * K + q], A[q], s);
      A[r] = s / C[r * K + r];
    }
    for (int r = k - 1; r >= 0; --r) {
      double s = A[r];
      for (int q = r + 1; q < k; ++q) s = fma(-C[q * K + r], A[q], s);
      A[r] = s / C[r * K + r];
    }
    double ar = 0.0, ac = 0.0;
    for (int i = 0; i < k; ++i) {
      if (a.r) ar += A[i] * a.r[N[i]];
      ac += A[i] * c[i];
    }
    if (a.mu_part) a.mu_part[p] = ar;
    if (a.laplace) {  // D_p = (s1 or r_q) - A.c, and A
      a.var_out[p] = (vif ? a.rq[p] : a.s1) - ac;
      for (int i = 0; i < K; ++i) a.A_out[static_cast<size_t>(p) * K + i] = i < k ? A[i] : 0.0;
    } else if (vif) {
      a.var_out[p] = a.rq[p] + a.sigma2 - ac;  // D_p
      for (int i = 0; i < K; ++i) a.A_out[static_cast<size_t>(p) * K + i] = i < k ? A[i] : 0.0;
    } else {
      const double v = a.s1 + a.sigma2 - ac;
      a.var_out[p] = v > 0.0 ? v : 0.0;
    }
  }
}

// Up(j, p) = k(z_j, q_p)
__global__ void target_cross_kernel(const double* zx, const double* zy, const int32_t* ztid, int M, int ldm,
                                    const double* qx, const double* qy, const int32_t* qtid, int np, DevKernel k,
                                    LagTable lt, double* Up) {
  for (int p = blockIdx.x; p < np; p += gridDim.x)
    for (int j = threadIdx.x; j < ldm; j += blockDim.x) {
      double v = 0.0;
      if (j < M) {
        double pe, pb;
        lt.get2(ztid[j], qtid[p], pe, pb);
        TF f;
        f.pow_mE = pe;
        f.pow_mbh = pb;
        v = gneiting_eval<true>(k, spatial_dist(zx[j], zy[j], qx[p], qy[p]), f);
      }
      Up[static_cast<size_t>(p) * ldm + j] = v;
    }
}

// per-column dot products: out[p] = sum_j A(j,p) B(j,p)
__global__ void coldot_kernel(int np, int ldm, const double* A, const double* B, double* out) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int p = gw; p < np; p += nw) {
    double s = 0.0;
    for (int j = lane; j < ldm; j += 32) s = fma(A[static_cast<size_t>(p) * ldm + j], B[static_cast<size_t>(p) * ldm + j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[p] = s;
  }
}

// W sN for each target: sum_a A_a W(:, N_a)
__global__ void wsn_kernel(int np, int m, int ldm, const int32_t* nbr, const double* A, const double* W, double* out) {
  for (int p = blockIdx.x; p < np; p += gridDim.x)
    for (int j = threadIdx.x; j < ldm; j += blockDim.x) {
      double s = 0.0;
      for (int a2 = 0; a2 < m; ++a2) {
        const int c = nbr[static_cast<size_t>(p) * m + a2];
        if (c < 0) break;
        s = fma(A[static_cast<size_t>(p) * m + a2], W[static_cast<size_t>(c) * ldm + j], s);
      }
      out[static_cast<size_t>(p) * ldm + j] = s;
    }
}

__global__ void resid_from_sq_kernel(int n, double s1, const double* sq, double* r) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) r[i] = s1 - sq[i];
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct TargetSet {
  DevBuf<double> qx, qy, qt;
  DevBuf<int32_t> qtid;
  std::vector<double> hx, hy, ht;
};

// Append the target times as a third time group and rebuild the lag tables.
static void setup_targets(stgp_structure* s, int np, const double* txyt, TargetSet& T) {
  stgp_ctx* ctx = s->ds->ctx;
  T.hx.resize(np);
  T.hy.resize(np);
  T.ht.resize(np);
  for (int p = 0; p < np; ++p) {
    T.hx[p] = txyt[3 * p];
    T.hy[p] = txyt[3 * p + 1];
    T.ht[p] = txyt[3 * p + 2];
    if (!std::isfinite(T.hx[p]) || !std::isfinite(T.hy[p]) || !std::isfinite(T.ht[p]))
      data_error("SpaceTimePoint: coordinates and time must be finite");
  }
  std::set<double> ts(T.ht.begin(), T.ht.end());
  std::vector<double> Tq(ts.begin(), ts.end());
  const int base = static_cast<int>(s->ti.T.size());
  std::vector<int32_t> qtid(np);
  for (int p = 0; p < np; ++p)
    qtid[p] = base + static_cast<int>(std::lower_bound(Tq.begin(), Tq.end(), T.ht[p]) - Tq.begin());
  TimeIndex ti = s->ti;
  ti.T.insert(ti.T.end(), Tq.begin(), Tq.end());
  ti.build();
  upload_lag_table(s->lt, ti, s->th, s->ds->lagpol, ctx->stream, true);
  s->ti_dirty = true;  // the structure's own index must be restored on the next build
  T.qx.upload(T.hx.data(), np, ctx->stream);
  T.qy.upload(T.hy.data(), np, ctx->stream);
  T.qt.upload(T.ht.data(), np, ctx->stream);
  T.qtid.upload(qtid.data(), np, ctx->stream);
}

static void target_neighbors(stgp_structure* s, TargetSet& T, int np, int pred_m_v, int metric, const double* Wq,
                             const double* rq, const double* resid, DevBuf<int32_t>& nbr, const double* wsq = nullptr,
                             const double* wqsq = nullptr) {
  stgp_ctx* ctx = s->ds->ctx;
  PredArgs a{};
  a.n = s->n;
  a.np = np;
  a.m = pred_m_v;
  a.x = s->ds->x.get();
  a.y = s->ds->y.get();
  a.t = s->ds->t.get();
  a.tid = s->ds->tid.get();
  a.qx = T.qx.get();
  a.qy = T.qy.get();
  a.qt = T.qt.get();
  a.qtid = T.qtid.get();
  a.metric = metric;
  a.ss = s->nbr_ss;
  a.ts = s->nbr_ts;
  a.k = dev_kernel(s->th);
  a.lt = lag_view(s->lt);
  a.s1 = s->th.sigma1_2;
  DevBuf<double> Td;
  if (s->ds->time_sorted) {
    Td.upload(s->ds->Tdata.data(), s->ds->Tdata.size(), ctx->stream);
    a.blk_start = s->ds->blk_start.get();
    a.Tdata = Td.get();
    a.nblk = static_cast<int>(s->ds->Tdata.size());
  }
  a.W = s->lr.W.get();
  a.ldm = s->lr.ldm;
  a.M = s->lr.M;
  a.resid = resid;
  a.Wq = Wq;
  a.rq = rq;
  DevBuf<double> brmin, bamax;
  if (metric == 2 && s->lr.M > 0 && wsq && wqsq) {
    a.wsq = wsq;
    a.wqsq = wqsq;
    if (a.blk_start) {
      brmin.alloc(static_cast<size_t>(a.nblk));
      bamax.alloc(static_cast<size_t>(a.nblk));
      block_bound_kernel<<<std::max(1, std::min(a.nblk, ctx->num_sms * 4)), 256, 0, ctx->stream>>>(
          a.nblk, a.blk_start, resid, wsq, s->th.sigma1_2, brmin.get(), bamax.get());
      launched(ctx);
      a.blk_rmin = brmin.get();
      a.blk_amax = bamax.get();
    }
  }
  nbr.ensure(static_cast<size_t>(np) * pred_m_v);
  a.nbr_out = nbr.get();
  DevBuf<double> scratch;
  if (pred_m_v <= 32) {
    target_knn_kernel<<<std::max(1, std::min(ceil_div(np, 8), ctx->num_sms * 8)), 256, 0, ctx->stream>>>(a);
  } else {
    scratch.alloc(static_cast<size_t>(np) * s->n);
    a.scratch_d = scratch.get();
    target_knn_generic_kernel<<<std::max(1, ceil_div(np, 64)), 64, 0, ctx->stream>>>(a);
  }
  launched(ctx);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
}

static void cond_solve(stgp_structure* s, TargetSet& T, int np, int pred_m_v, const DevBuf<int32_t>& nbr,
                       const double* rvec, bool vif, const double* Wq, const double* rq, double* mu_part, double* var,
                       double* Aout, bool laplace = false) {
  stgp_ctx* ctx = s->ds->ctx;
  CondArgs c{};
  c.np = np;
  c.m = pred_m_v;
  c.n = s->n;
  c.nbr = nbr.get();
  c.x = s->ds->x.get();
  c.y = s->ds->y.get();
  c.qx = T.qx.get();
  c.qy = T.qy.get();
  c.tid = s->ds->tid.get();
  c.qtid = T.qtid.get();
  c.k = dev_kernel(s->th);
  c.lt = lag_view(s->lt);
  c.s1 = s->th.sigma1_2;
  c.sigma2 = s->th.sigma2;
  c.r = rvec;
  c.W = s->lr.W.get();
  c.ldm = s->lr.ldm;
  c.M = vif ? s->lr.M : 0;
  c.Wq = Wq;
  c.rq = rq;
  c.mu_part = mu_part;
  c.var_out = var;
  c.A_out = Aout;
  c.laplace = laplace ? 1 : 0;
  if (laplace) c.sigma2 = 0.0;
  DevBuf<double> scratch(static_cast<size_t>(np) * (static_cast<size_t>(pred_m_v) * pred_m_v + 2 * pred_m_v));
  c.scratch = scratch.get();
  DevBuf<int> fail(1);
  fail.zero(ctx->stream);
  c.fail = fail.get();
  cond_solve_kernel<<<std::max(1, ceil_div(np, 64)), 64, 0, ctx->stream>>>(c, vif);
  launched(ctx);
  int f = 0;
  fail.download(&f, 1, ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (f && laplace)
    numeric_error(vif ? "VifLaplace: target conditioning block failed" : "VecchiaLaplace: target conditioning block failed");
  if (f)
    numeric_error(vif ? "predict: residual conditioning block not positive definite"
                      : "predict: conditioning block not positive definite");
}

// Vecchia (approximations.cpp:867-921)
void vecchia_predict(stgp_structure* s, int np, const double* txyt, int pred_m_v, double* mu, double* var) {
  stgp_ctx* ctx = s->ds->ctx;
  if (pred_m_v < 0) config_error("predict: pred_m_v must be >= 0");
  TargetSet T;
  setup_targets(s, np, txyt, T);
  const int metric = s->nbr_kind == STGP_METRIC_EUCLID ? 0 : 1;
  const int m = std::max(1, std::min(pred_m_v, s->n));
  DevBuf<int32_t> nbr;
  target_neighbors(s, T, np, m, metric, nullptr, nullptr, nullptr, nbr);
  DevBuf<double> mp(np), vp(np);
  cond_solve(s, T, np, m, nbr, s->r.get(), false, nullptr, nullptr, mp.get(), vp.get(), nullptr);
  mp.download(mu, np, ctx->stream);
  vp.download(var, np, ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
}

static void fitc_predict(stgp_structure* s, TargetSet& T, int np, double* mu, double* var) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, ldm = L.ldm;
  cudaStream_t st = ctx->stream;
  // alpha = rl - Lambda^{-1} W^T K^{-1} W rl;  Walpha = W alpha
  std::unique_ptr<ProfRegion> pr(new ProfRegion(ctx, "p_alpha"));
  double* rl = L.tmp("p_rl", n);
  double* kv = L.tmp("p_kv", ldm);
  double* t = L.tmp("p_t", n);
  double* alpha = L.tmp("p_alpha", n);
  div_vec(ctx, n, s->r.get(), L.lambda.get(), rl);
  dev_gemv(ctx, false, ldm, n, 1.0, L.W.get(), ldm, rl, 0.0, kv);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, false);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, true);
  dev_gemv(ctx, true, ldm, n, 1.0, L.W.get(), ldm, kv, 0.0, t);
  div_vec(ctx, n, t, L.lambda.get(), t);
  vsub(ctx, n, rl, t, alpha);
  double* walpha = L.tmp("p_walpha", ldm);
  dev_gemv(ctx, false, ldm, n, 1.0, L.W.get(), ldm, alpha, 0.0, walpha);
  // targets: Up, What = L_m^{-1} Up, Y = L_K^{-1} What
  pr.reset(new ProfRegion(ctx, "p_targets"));
  DevBuf<double> Up(static_cast<size_t>(ldm) * np), Wh(static_cast<size_t>(ldm) * np), Y(static_cast<size_t>(ldm) * np);
  target_cross_kernel<<<std::max(1, std::min(np, ctx->num_sms * 8)), 128, 0, st>>>(
      L.zx.get(), L.zy.get(), L.ztid.get(), L.M, ldm, T.qx.get(), T.qy.get(), T.qtid.get(), np, dev_kernel(s->th),
      lag_view(s->lt), Up.get());
  launched(ctx);
  dev_trmm_left(ctx, L.Lminv.get(), ldm, ldm, Up.get(), ldm, np, false, Wh.get(), ldm);
  STGP_CUDA(cudaMemcpyAsync(Y.get(), Wh.get(), sizeof(double) * ldm * np, cudaMemcpyDeviceToDevice, st));
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, Y.get(), ldm, np, false);
  DevBuf<double> mu_d(np), w2(np), y2(np);
  dev_gemv(ctx, true, ldm, np, 1.0, Wh.get(), ldm, walpha, 0.0, mu_d.get());
  coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, ldm, Wh.get(), Wh.get(), w2.get());
  launched(ctx);
  coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, ldm, Y.get(), Y.get(), y2.get());
  launched(ctx);
  pr.reset();
  std::vector<double> hw(np), hy(np);
  mu_d.download(mu, np, st);
  w2.download(hw.data(), np, st);
  y2.download(hy.data(), np, st);
  STGP_CUDA(cudaStreamSynchronize(st));
  for (int p = 0; p < np; ++p) {
    // shrink = wp'(A1 - A2) wp = |What|^2 - |L_K^{-1} What|^2 (approximations.cpp:950-955)
    const double v = s->th.sigma1_2 + s->th.sigma2 - (hw[p] - hy[p]);
    var[p] = v > 0.0 ? v : 0.0;
  }
}

static void vif_predict(stgp_structure* s, TargetSet& T, int np, int pred_m_v, double* mu, double* var) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, M = L.M, ldm = L.ldm;
  cudaStream_t st = ctx->stream;
  // z = r - t and W alpha = V' D^{-1} B z (alpha = Q z)
  double* z = L.tmp("p_z", n);
  double* Bz = L.tmp("p_Bz", n);
  double* walpha = L.tmp("p_walpha", ldm);
  if (M > 0) {
    const int nb = std::max(1, std::min(ceil_div(n, 256), ctx->num_sms * 4));
    s->red.ensure(nb, 1);
    s->u.ensure(n);
    launch_nll_stored(s, nb, s->u.get());
    double* g1 = L.tmp("p_g1", n);
    double* yhat = L.tmp("p_yhat", ldm);
    double* t = L.tmp("p_t", n);
    div_vec(ctx, n, s->u.get(), s->D.get(), g1);
    dev_gemv(ctx, false, ldm, n, 1.0, L.Vp.get(), ldm, g1, 0.0, yhat);
    dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, yhat, ldm, 1, false);
    dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, yhat, ldm, 1, true);
    dev_gemv(ctx, true, ldm, n, 1.0, L.W.get(), ldm, yhat, 0.0, t);
    vsub(ctx, n, s->r.get(), t, z);
    b_apply(s, z, Bz);
    div_vec(ctx, n, Bz, s->D.get(), Bz);
    dev_gemv(ctx, false, ldm, n, 1.0, L.Vp.get(), ldm, Bz, 0.0, walpha);
  } else {
    STGP_CUDA(cudaMemcpyAsync(z, s->r.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  // targets: up, wq = L_m^{-1} up, r_q = s1 - |wq|^2; training residual variances
  DevBuf<double> Up(static_cast<size_t>(ldm) * np), Wq(static_cast<size_t>(ldm) * np), rq(np), wq2(np);
  double* resid = L.tmp("p_resid", n);
  if (M > 0) {
    target_cross_kernel<<<std::max(1, std::min(np, ctx->num_sms * 8)), 128, 0, st>>>(
        L.zx.get(), L.zy.get(), L.ztid.get(), M, ldm, T.qx.get(), T.qy.get(), T.qtid.get(), np, dev_kernel(s->th),
        lag_view(s->lt), Up.get());
    launched(ctx);
    dev_trmm_left(ctx, L.Lminv.get(), ldm, ldm, Up.get(), ldm, np, false, Wq.get(), ldm);
    coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, ldm, Wq.get(), Wq.get(), wq2.get());
    launched(ctx);
    resid_from_sq_kernel<<<grid_for(np), 256, 0, st>>>(np, s->th.sigma1_2, wq2.get(), rq.get());
    launched(ctx);
    double* sq = L.tmp("p_sq", n);
    coldot_kernel<<<grid_for(static_cast<long long>(n) * 32), 256, 0, st>>>(n, ldm, L.W.get(), L.W.get(), sq);
    launched(ctx);
    resid_from_sq_kernel<<<grid_for(n), 256, 0, st>>>(n, s->th.sigma1_2, sq, resid);
    launched(ctx);
  } else {
    std::vector<double> s1v(std::max(n, np), s->th.sigma1_2);
    STGP_CUDA(cudaMemcpyAsync(rq.get(), s1v.data(), sizeof(double) * np, cudaMemcpyHostToDevice, st));
    STGP_CUDA(cudaMemcpyAsync(resid, s1v.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    STGP_CUDA(cudaMemsetAsync(wq2.get(), 0, sizeof(double) * np, st));
  }
  const int m = std::max(1, std::min(pred_m_v, n));
  DevBuf<int32_t> nbr;
  target_neighbors(s, T, np, m, 2, Wq.get(), rq.get(), resid, nbr, M > 0 ? L.tmp("p_sq", n) : nullptr,
                   M > 0 ? wq2.get() : nullptr);
  DevBuf<double> mp(np), Dp(np), A(static_cast<size_t>(np) * m);
  cond_solve(s, T, np, m, nbr, z, true, Wq.get(), rq.get(), mp.get(), Dp.get(), A.get());
  std::vector<double> hmu(np), hD(np), hwq2(np), hwa(np, 0.0), hcross(np, 0.0), hq(np, 0.0), hh(np, 0.0);
  mp.download(hmu.data(), np, st);
  Dp.download(hD.data(), np, st);
  wq2.download(hwq2.data(), np, st);
  if (M > 0) {
    DevBuf<double> Wsn(static_cast<size_t>(ldm) * np), KW(static_cast<size_t>(ldm) * np), H(static_cast<size_t>(ldm) * np),
        d1(np), d2(np), d3(np), d4(np);
    wsn_kernel<<<std::max(1, std::min(np, ctx->num_sms * 8)), 128, 0, st>>>(np, m, ldm, nbr.get(), A.get(), L.W.get(),
                                                                            Wsn.get());
    launched(ctx);
    // (K - I) wq = K wq - wq
    dev_gemm(ctx, false, false, ldm, np, ldm, 1.0, L.Kfull.get(), ldm, Wq.get(), ldm, 0.0, KW.get(), ldm);
    vsub(ctx, static_cast<long long>(ldm) * np, KW.get(), Wq.get(), KW.get());
    // h = W sN + (K - I) wq ; |L_K^{-1} h|^2 = h' K^{-1} h
    vadd(ctx, static_cast<long long>(ldm) * np, Wsn.get(), KW.get(), H.get());
    dev_gemv(ctx, true, ldm, np, 1.0, Wq.get(), ldm, walpha, 0.0, d4.get());
    coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, ldm, Wq.get(), Wsn.get(), d1.get());
    launched(ctx);
    coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, ldm, Wq.get(), KW.get(), d2.get());
    launched(ctx);
    dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, H.get(), ldm, np, false);
    coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, ldm, H.get(), H.get(), d3.get());
    launched(ctx);
    d1.download(hcross.data(), np, st);
    d2.download(hq.data(), np, st);
    d3.download(hh.data(), np, st);
    d4.download(hwa.data(), np, st);
  }
  STGP_CUDA(cudaStreamSynchronize(st));
  for (int p = 0; p < np; ++p) {
    mu[p] = hwa[p] + hmu[p];
    const double v = hwq2[p] + hD[p] - 2.0 * hcross[p] - hq[p] + hh[p];
    var[p] = v > 0.0 ? v : 0.0;
  }
}


// ---------------------------------------------------------------------------
// ZC-PTN prediction (laplace.cpp:205-259) on the Laplace state at the mode: latent cross covariances
// k_p (the LaplaceAlgebra target rows, approximations.cpp:1121-1160, 1202-1215, 1290-1355), then
//   mu_p = x_p beta + k_p . a,   var_p = k_pp - k_p' W k_p + (W k_p)' (Sigma^{-1} + W)^{-1} (W k_p),
// for all targets at once (n x n_p matrices).  For Vecchia / VIF, Sigma_s s_N = B^{-1} D B^{-T} s_N is
// two triangular solves with the dense unit-lower B.
// ---------------------------------------------------------------------------
namespace {
__global__ void dense_b_kernel(int n, int m_v, const int32_t* nbr, const double* A, double* B) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    B[static_cast<size_t>(i) * n + i] = 1.0;
    for (int a = 0; a < m_v; ++a) {
      const int j = nbr[static_cast<size_t>(i) * m_v + a];
      if (j >= 0) B[static_cast<size_t>(j) * n + i] = -A[static_cast<size_t>(i) * m_v + a];
    }
  }
}
// SN(:, p) = A_p scattered at the target's neighbours
__global__ void scatter_sn_kernel(int n, int np, int m, const int32_t* nbr, const double* A, double* SN) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x)
    for (int a = 0; a < m; ++a) {
      const int j = nbr[static_cast<size_t>(p) * m + a];
      if (j >= 0) SN[static_cast<size_t>(p) * n + j] = A[static_cast<size_t>(p) * m + a];
    }
}
__global__ void scale_rows_kernel(int n, long long ncols, const double* d, double* X) {
  const long long total = static_cast<long long>(n) * ncols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    X[e] *= d[e % n];
}
// var_prior(p) = base(p) + D_p + sum_a A_p[a] Kp(N_p[a], p)
__global__ void prior_var_kernel(int n, int np, int m, const int32_t* nbr, const double* A, const double* Kp,
                                 const double* Dp, const double* base, double* out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
    double v = (base ? base[p] : 0.0) + Dp[p];
    for (int a = 0; a < m; ++a) {
      const int j = nbr[static_cast<size_t>(p) * m + a];
      if (j >= 0) v += A[static_cast<size_t>(p) * m + a] * Kp[static_cast<size_t>(p) * n + j];
    }
    out[p] = v;
  }
}
}  // namespace

void zcptn_moments_dev(stgp_structure* s, const double* a_host, const double* w_host, int np, const double* txyt,
                       int pred_m_v, double* mu_lat, double* var_lat) {
  stgp_ctx* ctx = s->ds->ctx;
  cudaStream_t st = ctx->stream;
  const int n = s->n;
  LowRank& L = s->lr;
  const int ldm = L.ldm, M = s->kind == STGP_VECCHIA ? 0 : L.M;
  if (pred_m_v < 0) config_error("predict: pred_m_v must be >= 0");
  if (s->kind != STGP_FITC && n > 40000)
    config_error("Laplace algebra: the dense factorization of Q + W supports n <= 40000 (desk scale, SPEC.md:9)");
  DevBuf<double> wv(n), av(n);
  wv.upload(w_host, n, st);
  av.upload(a_host, n, st);
  laplace_prepare_w(s, wv.get());
  TargetSet T;
  setup_targets(s, np, txyt, T);
  DevBuf<double> Kp(static_cast<size_t>(n) * np), kpp(np);
  DevBuf<double> Up, Wq;
  if (M > 0) {
    Up.alloc(static_cast<size_t>(ldm) * np);
    Wq.alloc(static_cast<size_t>(ldm) * np);
    target_cross_kernel<<<std::max(1, std::min(np, ctx->num_sms * 8)), 128, 0, st>>>(
        L.zx.get(), L.zy.get(), L.ztid.get(), M, ldm, T.qx.get(), T.qy.get(), T.qtid.get(), np, dev_kernel(s->th),
        lag_view(s->lt), Up.get());
    launched(ctx);
    dev_trmm_left(ctx, L.Lminv.get(), ldm, ldm, Up.get(), ldm, np, false, Wq.get(), ldm);  // w_q = L_m^{-1} u_p
  }
  if (s->kind == STGP_FITC) {  // k_p = U^T Sigma_m^{-1} u_p = W^T w_q, k_pp = s1
    dev_gemm(ctx, true, false, n, np, ldm, 1.0, L.W.get(), ldm, Wq.get(), ldm, 0.0, Kp.get(), n);
    std::vector<double> s1v(np, s->th.sigma1_2);
    kpp.upload(s1v.data(), np, st);
  } else {
    const bool vif = s->kind == STGP_VIF;
    DevBuf<double> rq(np), wq2(np);
    double* resid = nullptr;
    if (vif && M > 0) {
      coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, ldm, Wq.get(), Wq.get(), wq2.get());
      launched(ctx);
      resid_from_sq_kernel<<<grid_for(np), 256, 0, st>>>(np, s->th.sigma1_2, wq2.get(), rq.get());
      launched(ctx);
      double* sq = L.tmp("p_sq", n);
      coldot_kernel<<<grid_for(static_cast<long long>(n) * 32), 256, 0, st>>>(n, ldm, L.W.get(), L.W.get(), sq);
      launched(ctx);
      resid = L.tmp("p_resid", n);
      resid_from_sq_kernel<<<grid_for(n), 256, 0, st>>>(n, s->th.sigma1_2, sq, resid);
      launched(ctx);
    } else if (vif) {
      std::vector<double> s1v(std::max(n, np), s->th.sigma1_2);
      resid = L.tmp("p_resid", n);
      STGP_CUDA(cudaMemcpyAsync(rq.get(), s1v.data(), sizeof(double) * np, cudaMemcpyHostToDevice, st));
      STGP_CUDA(cudaMemcpyAsync(resid, s1v.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
      STGP_CUDA(cudaMemsetAsync(wq2.get(), 0, sizeof(double) * np, st));
    }
    const int m = std::max(1, std::min(pred_m_v, n));
    DevBuf<int32_t> nbr;
    if (vif)
      target_neighbors(s, T, np, m, 2, M > 0 ? Wq.get() : nullptr, rq.get(), resid, nbr, M > 0 ? L.tmp("p_sq", n) : nullptr,
                       M > 0 ? wq2.get() : nullptr);
    else
      target_neighbors(s, T, np, m, s->nbr_kind == STGP_METRIC_EUCLID ? 0 : 1, nullptr, nullptr, nullptr, nbr);
    DevBuf<double> Dp(np), A(static_cast<size_t>(np) * m);
    cond_solve(s, T, np, m, nbr, nullptr, vif, M > 0 ? Wq.get() : nullptr, vif ? rq.get() : nullptr, nullptr, Dp.get(),
               A.get(), true);
    // Kp = Sigma_s SN = B^{-1} D B^{-T} SN
    DevBuf<double> Bd(static_cast<size_t>(n) * n);
    Bd.zero(st);
    dense_b_kernel<<<grid_for(n), 256, 0, st>>>(n, s->m_v, s->nbr.get(), s->A.get(), Bd.get());
    launched(ctx);
    Kp.zero(st);
    scatter_sn_kernel<<<grid_for(np), 256, 0, st>>>(n, np, m, nbr.get(), A.get(), Kp.get());
    launched(ctx);
    dev_trsm_left(ctx, Bd.get(), n, n, Kp.get(), n, np, true);
    scale_rows_kernel<<<grid_for(static_cast<long long>(n) * np), 256, 0, st>>>(n, np, s->D.get(), Kp.get());
    launched(ctx);
    dev_trsm_left(ctx, Bd.get(), n, n, Kp.get(), n, np, false);
    prior_var_kernel<<<grid_for(np), 256, 0, st>>>(n, np, m, nbr.get(), A.get(), Kp.get(), Dp.get(),
                                                   vif && M > 0 ? wq2.get() : nullptr, kpp.get());
    launched(ctx);
    if (vif && M > 0)  // + U^T Sigma_m^{-1} u_p = W^T w_q
      dev_gemm(ctx, true, false, n, np, ldm, 1.0, L.W.get(), ldm, Wq.get(), ldm, 1.0, Kp.get(), n);
  }
  // mu = k . a ; var = k_pp - k' W k + (W k)' (Sigma^{-1} + W)^{-1} (W k)
  DevBuf<double> muv(np), q1(np), q2(np), WK(static_cast<size_t>(n) * np), SW(static_cast<size_t>(n) * np);
  dev_gemv(ctx, true, n, np, 1.0, Kp.get(), n, av.get(), 0.0, muv.get());
  STGP_CUDA(cudaMemcpyAsync(WK.get(), Kp.get(), sizeof(double) * n * np, cudaMemcpyDeviceToDevice, st));
  scale_rows_kernel<<<grid_for(static_cast<long long>(n) * np), 256, 0, st>>>(n, np, wv.get(), WK.get());
  launched(ctx);
  coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, n, Kp.get(), WK.get(), q1.get());
  launched(ctx);
  laplace_solve_cols(s, WK.get(), np, SW.get());
  coldot_kernel<<<grid_for(static_cast<long long>(np) * 32), 256, 0, st>>>(np, n, WK.get(), SW.get(), q2.get());
  launched(ctx);
  std::vector<double> hk(np), h1(np), h2(np);
  muv.download(mu_lat, np, st);
  kpp.download(hk.data(), np, st);
  q1.download(h1.data(), np, st);
  q2.download(h2.data(), np, st);
  STGP_CUDA(cudaStreamSynchronize(st));
  for (int p = 0; p < np; ++p) var_lat[p] = std::max(hk[p] - h1[p] + h2[p], 0.0);
}

void lowrank_predict(stgp_structure* s, int np, const double* txyt, int pred_m_v, double* mu, double* var) {
  TargetSet T;
  setup_targets(s, np, txyt, T);
  if (s->kind == STGP_FITC) {
    fitc_predict(s, T, np, mu, var);
  } else {
    if (pred_m_v < 0) config_error("predict: pred_m_v must be >= 0");
    vif_predict(s, T, np, pred_m_v, mu, var);
  }
}

// Sigma~^{-1} v on the device (approximations.cpp:769-798)
void sigma_inv_apply_dev(stgp_structure* s, const double* v, double* out) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, ldm = L.ldm;
  if (s->kind == STGP_VECCHIA || (s->kind == STGP_VIF && L.M == 0)) {
    double* u = L.tmp("g_u", n);
    b_apply(s, v, u);
    div_vec(ctx, n, u, s->D.get(), u);
    bt_apply(s, u, out);
    return;
  }
  double* kv = L.tmp("g_kv", ldm);
  if (s->kind == STGP_FITC) {
    double* vl = L.tmp("g_vl", n);
    double* t = L.tmp("g_t", n);
    div_vec(ctx, n, v, L.lambda.get(), vl);
    dev_gemv(ctx, false, ldm, n, 1.0, L.W.get(), ldm, vl, 0.0, kv);
    dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, false);
    dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, true);
    dev_gemv(ctx, true, ldm, n, 1.0, L.W.get(), ldm, kv, 0.0, t);
    div_vec(ctx, n, t, L.lambda.get(), t);
    vsub(ctx, n, vl, t, out);
    return;
  }
  // VIF: Q v - Q W^T K^{-1} W Q v, with W Q v = V' D^{-1} B v
  double* u = L.tmp("g_u", n);
  double* qv = L.tmp("g_qv", n);
  double* t = L.tmp("g_t", n);
  b_apply(s, v, u);
  div_vec(ctx, n, u, s->D.get(), u);
  bt_apply(s, u, qv);
  dev_gemv(ctx, false, ldm, n, 1.0, L.Vp.get(), ldm, u, 0.0, kv);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, false);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, kv, ldm, 1, true);
  dev_gemv(ctx, true, ldm, n, 1.0, L.W.get(), ldm, kv, 0.0, t);
  b_apply(s, t, u);
  div_vec(ctx, n, u, s->D.get(), u);
  bt_apply(s, u, t);
  vsub(ctx, n, qv, t, out);
}

// gls_from_solver (approximations.cpp:752-765): device Sigma~^{-1} X_j, device dots, host p x p solve
void gls_beta_device(stgp_structure* s, const double* y_host, const double* X_host, int p, double* beta_out) {
  stgp_ctx* ctx = s->ds->ctx;
  const int n = s->n;
  const double *Xd, *yd;
  if (y_host) {
    s->Xwork.upload(X_host, static_cast<size_t>(n) * p, ctx->stream);
    s->ywork.upload(y_host, static_cast<size_t>(n), ctx->stream);
    Xd = s->Xwork.get();
    yd = s->ywork.get();
  } else {
    if (!s->ds->has_resp || s->ds->p != p) config_error("gls_beta: resident covariates do not match p");
    Xd = s->ds->X.get();
    yd = s->ds->resp.get();
  }
  DevBuf<double> SX(static_cast<size_t>(n) * p);
  for (int j = 0; j < p; ++j) sigma_inv_apply_dev(s, Xd + static_cast<size_t>(j) * n, SX.get() + static_cast<size_t>(j) * n);
  std::vector<double> A(static_cast<size_t>(p) * p), b(static_cast<size_t>(p));
  Reducer red;
  for (int j = 0; j < p; ++j) {
    for (int a = 0; a < p; ++a)
      A[static_cast<size_t>(a) + static_cast<size_t>(j) * p] =
          dev_dot(ctx, Xd + static_cast<size_t>(a) * n, SX.get() + static_cast<size_t>(j) * n, n, red);
    b[static_cast<size_t>(j)] = dev_dot(ctx, SX.get() + static_cast<size_t>(j) * n, yd, n, red);
  }
  // p x p symmetric positive definite solve (LDLT in the reference)
  std::vector<double> Lf(A);
  for (int j = 0; j < p; ++j) {
    double d = Lf[static_cast<size_t>(j) * p + j];
    for (int k = 0; k < j; ++k) d -= Lf[static_cast<size_t>(j) + static_cast<size_t>(k) * p] * Lf[static_cast<size_t>(j) + static_cast<size_t>(k) * p];
    if (!(d > 0.0)) numeric_error("gls_beta: normal equations are singular");
    d = std::sqrt(d);
    Lf[static_cast<size_t>(j) + static_cast<size_t>(j) * p] = d;
    for (int r = j + 1; r < p; ++r) {
      double v = Lf[static_cast<size_t>(r) + static_cast<size_t>(j) * p];
      for (int k = 0; k < j; ++k) v -= Lf[static_cast<size_t>(r) + static_cast<size_t>(k) * p] * Lf[static_cast<size_t>(j) + static_cast<size_t>(k) * p];
      Lf[static_cast<size_t>(r) + static_cast<size_t>(j) * p] = v / d;
    }
  }
  std::vector<double> zv(b);
  for (int r = 0; r < p; ++r) {
    for (int k = 0; k < r; ++k) zv[static_cast<size_t>(r)] -= Lf[static_cast<size_t>(r) + static_cast<size_t>(k) * p] * zv[static_cast<size_t>(k)];
    zv[static_cast<size_t>(r)] /= Lf[static_cast<size_t>(r) + static_cast<size_t>(r) * p];
  }
  for (int r = p - 1; r >= 0; --r) {
    for (int k = r + 1; k < p; ++k) zv[static_cast<size_t>(r)] -= Lf[static_cast<size_t>(k) + static_cast<size_t>(r) * p] * zv[static_cast<size_t>(k)];
    zv[static_cast<size_t>(r)] /= Lf[static_cast<size_t>(r) + static_cast<size_t>(r) * p];
  }
  std::copy(zv.begin(), zv.end(), beta_out);
}

}  // namespace stgp

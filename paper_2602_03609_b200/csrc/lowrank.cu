// FITC / VIF low-rank algebra (approximations.cpp:217-312, 352-384, 495-744).
//
// Everything is carried in the whitened basis of the inducing Cholesky factor
// L_m (Sigma_m + jitter = L_m L_m^T, inducing.cpp:237-262):
//   W = L_m^{-1} U            (U_ji = k(z_j, p_i), M x n)
//   VIF:  V' = W B^T,  K = I + V' D^{-1} V'^T  so that M_core = L_m K L_m^T and
//         log|M_core| - log|Sigma_m| = log|K|, w' M^{-1} w = (W ur)' K^{-1} (W ur)
//   FITC: K = I + W Lambda^{-1} W^T
// The reference's M x n temporaries (P = Sigma_m^{-1} U, N1, Hhat, omega, ...)
// become L_m^{-T} times whitened quantities; the only dense n x M^2 work left is
// the TRSM for W, one SYRK for K, two TRSMs for X = K^{-1} V', one GEMM for the
// Sigma_m-pair weights and one TRSM for omega -- the canonical 3.5 n M^2 of
// SURVEY.md §8(d).  All sparse B / B^T products are deterministic gathers (a
// CSC of B's pattern is built once per structure).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <set>

#include <cub/device/device_scan.cuh>

#include "comm.hpp"
#include "dense.cuh"
#include "lowrank_common.cuh"
#include "ozaki.cuh"
#include "rows.cuh"
#include "structure.hpp"
#include "../../include/stgp_b200.h"

namespace stgp {

namespace {

constexpr int kT = kLrThreads;
constexpr int kMaxGatherM = 512;  // neighbour-set width supported by the column gathers

struct ZPts {
  const double *zx, *zy;
  const int32_t* ztid;
};

// Sigma_m(i, j) = k(z_i, z_j) (inducing.cpp:242-249) + diagonal jitter; padded part = identity
__global__ void sigma_m_kernel(ZPts z, int M, int ldm, DevKernel k, LagTable lt, double jit1, double jit2,
                               double* S) {
  const long long total = static_cast<long long>(ldm) * ldm;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e % ldm), c = static_cast<int>(e / ldm);
    double v;
    if (r >= M || c >= M) {
      v = r == c ? 1.0 : 0.0;
    } else {
      const int a = r >= c ? r : c, b = r >= c ? c : r;  // evaluate k(z_a, z_b), a >= b (loop order of the reference)
      double pe, pb;
      lt.get2(z.ztid[a], z.ztid[b], pe, pb);
      TF f;
      f.pow_mE = pe;
      f.pow_mbh = pb;
      v = gneiting_eval<true>(k, spatial_dist(z.zx[a], z.zy[a], z.zx[b], z.zy[b]), f);
      if (r == c) {
        v = __dadd_rn(v, jit1);
        if (jit2 != 0.0) v = __dadd_rn(v, jit2);
      }
    }
    S[static_cast<size_t>(c) * ldm + r] = v;
  }
}

// U(j, i) = k(z_j, p_i) (approximations.cpp:226-232), columns [c0, c1)
template <bool GEN>
__global__ void cross_cov_kernel(ZPts z, int M, int ldm, const double* x, const double* y, const int32_t* tid,
                                 int c0, int c1, DevKernel k, LagTable lt, double* U) {
  for (int i = c0 + blockIdx.x; i < c1; i += gridDim.x) {
    const double xi = x[i], yi = y[i];
    const int ti = tid[i];
    double* col = U + static_cast<size_t>(i) * ldm;
    for (int j = threadIdx.x; j < ldm; j += blockDim.x) {
      double v = 0.0;
      if (j < M) {
        double pe, pb;
        lt.get2(z.ztid[j], ti, pe, pb);
        TF f;
        f.pow_mE = pe;
        f.pow_mbh = pb;
        v = gneiting_eval<GEN>(k, spatial_dist(z.zx[j], z.zy[j], xi, yi), f);
      }
      col[j] = v;
    }
  }
}

// V'(:, r) = (W B^T)(:, r) = W(:, r) - sum_a A(r, a) W(:, N_a)   (approximations.cpp:298-305)
// The neighbour count is fixed before the j loop so the m_v column loads are batched (unrolled)
// rather than serialised behind a data-dependent exit.
__global__ void __launch_bounds__(128) vprime_kernel(const double* W, int ldm, const int32_t* nbr, int m_v,
                                                     const double* A, int r0, int r1, const int32_t* order,
                                                     unsigned long long* next, double* Vp) {
  __shared__ int sN[kMaxGatherM];
  __shared__ double sA[kMaxGatherM];
  __shared__ int sk, s_kr;
  for (;;) {  // rows claimed in order (claim_next): the in-flight rows stay a contiguous window
    __syncthreads();
    if (threadIdx.x == 0) {
      s_kr = static_cast<int>(atomicAdd(next, 1ull));
      sk = m_v;
    }
    __syncthreads();
    const int kr = s_kr;
    if (kr >= r1 - r0) break;
    const int r = order ? order[kr] : r0 + kr;
    for (int a = threadIdx.x; a < m_v; a += blockDim.x) {
      const int c = nbr[static_cast<size_t>(r) * m_v + a];
      sN[a] = c;
      sA[a] = A[static_cast<size_t>(r) * m_v + a];
      if (c < 0 && (a == 0 || nbr[static_cast<size_t>(r) * m_v + a - 1] >= 0)) sk = a;  // packed: first -1
    }
    __syncthreads();
    const int k = sk;
    for (int j = threadIdx.x; j < ldm; j += blockDim.x) {
      double acc = 0.0;
#pragma unroll 8
      for (int a = 0; a < k; ++a) acc += -sA[a] * __ldg(&W[static_cast<size_t>(sN[a]) * ldm + j]);
      acc += W[static_cast<size_t>(r) * ldm + j];
      Vp[static_cast<size_t>(r) * ldm + j] = acc;
    }
  }
}

// out(:, i) = in(:, i) * s_i
__global__ void scale_cols_kernel(const double* in, int ldm, long long ncols, const double* s, bool rsqrt_of,
                                  double* out) {
  const long long total = static_cast<long long>(ldm) * ncols;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / ldm;
    const double f = rsqrt_of ? 1.0 / sqrt(s[i]) : s[i];
    out[e] = in[e] * f;
  }
}

__global__ void set_identity_kernel(double* A, int ld, int n) {
  const long long total = static_cast<long long>(ld) * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    A[e] = (e % ld == e / ld) ? 1.0 : 0.0;
}

__global__ void vsub_kernel(long long n, const double* a, const double* b, double* out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = a[i] - b[i];
}
__global__ void vadd_kernel(long long n, const double* a, const double* b, double* out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = a[i] + b[i];
}

// y = a * x (+ b * z) elementwise helpers
__global__ void axpby_kernel(int n, double a, const double* x, double b, const double* z, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[i] = a * x[i] + (z ? b * z[i] : 0.0);
}
__global__ void div_kernel(int n, const double* x, const double* d, double* y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = x[i] / d[i];
}

// (B v)_i = v_i - sum_a A(i, a) v_{N_a}
__global__ void b_apply_kernel(int r0, int r1, int m_v, const int32_t* nbr, const double* A, const double* v,
                               double* out) {
  for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int a = 0; a < m_v; ++a) {
      const int j = nbr[static_cast<size_t>(i) * m_v + a];
      if (j < 0) break;
      s += -A[static_cast<size_t>(i) * m_v + a] * v[j];
    }
    out[i] = s + v[i];
  }
}

// CSC of B's pattern: column j lists (row r, slot) with N_r[slot] == j, plus (j, -1) for the diagonal.
__global__ void csc_count_kernel(int n, int m_v, const int32_t* nbr, int32_t* cnt) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(n) * m_v;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int j = nbr[e];
    if (j >= 0) atomicAdd(&cnt[j], 1);
  }
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) atomicAdd(&cnt[j], 1);
}
__global__ void csc_fill_kernel(int n, int m_v, const int32_t* nbr, const int32_t* ptr, int32_t* fillc, int32_t* erow,
                                int16_t* eslot) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       e < static_cast<long long>(n) * (m_v + 1); e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / (m_v + 1));
    const int a = static_cast<int>(e % (m_v + 1));
    int j;
    if (a == m_v) {
      j = r;
    } else {
      j = nbr[static_cast<size_t>(r) * m_v + a];
      if (j < 0) continue;
    }
    const int pos = ptr[j] + atomicAdd(&fillc[j], 1);
    erow[pos] = r;
    eslot[pos] = static_cast<int16_t>(a == m_v ? -1 : a);
  }
}
// sort each column's entries by row (insertion sort; columns hold ~m_v + 1 entries)
__global__ void csc_sort_kernel(int n, const int32_t* ptr, int32_t* erow, int16_t* eslot) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int b = ptr[j], e = ptr[j + 1];
    for (int p = b + 1; p < e; ++p) {
      const int r = erow[p];
      const int16_t s = eslot[p];
      int q = p - 1;
      while (q >= b && erow[q] > r) {
        erow[q + 1] = erow[q];
        eslot[q + 1] = eslot[q];
        --q;
      }
      erow[q + 1] = r;
      eslot[q + 1] = s;
    }
  }
}

// (B^T v)_j = sum over column j entries of B(r, j) v_r (deterministic, rows ascending)
__global__ void bt_apply_kernel(int c0, int c1, int m_v, const int32_t* ptr, const int32_t* erow, const int16_t* eslot,
                                const double* A, const double* v, double* out) {
  for (int j = c0 + blockIdx.x * blockDim.x + threadIdx.x; j < c1; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int p = ptr[j]; p < ptr[j + 1]; ++p) {
      const int r = erow[p];
      const int sl = eslot[p];
      const double b = sl < 0 ? 1.0 : -A[static_cast<size_t>(r) * m_v + sl];
      s += b * v[r];
    }
    out[j] = s;
  }
}

// E_r = X_r / D_r - 2 c0_r V'_r + Zr_r - yhat (Bz)_r / D_r and F_r = c0_r V'_r - Zr_r with
// Zr_r = sum_a Rv_r[a] W_{N_a} (E overwrites X in place: column r of X is read only here).
// The yhat term folds yM (ur - Q t)^T of the reference row by row: ur - Q t = Q z = B^T D^{-1} B z.
__global__ void __launch_bounds__(128) ef_kernel(int r0, int r1, int ldm, int m_v, const int32_t* nbr,
                                                 const double* Rv, const double* c0, const double* D, const double* W,
                                                 const double* Vp, const double* yhat, const double* Bz,
                                                 const int32_t* order, unsigned long long* next, double* X_E,
                                                 double* F) {
  __shared__ int sN[kMaxGatherM];
  __shared__ double sR[kMaxGatherM];
  __shared__ int sk, s_kr;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_kr = static_cast<int>(atomicAdd(next, 1ull));
      sk = m_v;
    }
    __syncthreads();
    const int kr = s_kr;
    if (kr >= r1 - r0) break;
    const int r = order ? order[kr] : r0 + kr;
    for (int a = threadIdx.x; a < m_v; a += blockDim.x) {
      const int c = nbr[static_cast<size_t>(r) * m_v + a];
      sN[a] = c;
      sR[a] = Rv[static_cast<size_t>(r) * m_v + a];
      if (c < 0 && (a == 0 || nbr[static_cast<size_t>(r) * m_v + a - 1] >= 0)) sk = a;
    }
    __syncthreads();
    const int k = sk;
    const double cr = c0[r], inv = 1.0 / D[r], qr = Bz[r] * inv;
    for (int j = threadIdx.x; j < ldm; j += blockDim.x) {
      double zr = 0.0;
#pragma unroll 8
      for (int a = 0; a < k; ++a) zr = fma(sR[a], __ldg(&W[static_cast<size_t>(sN[a]) * ldm + j]), zr);
      const size_t o = static_cast<size_t>(r) * ldm + j;
      const double v = Vp[o];
      X_E[o] = X_E[o] * inv - 2.0 * cr * v + zr - yhat[j] * qr;
      F[o] = cr * v - zr;
    }
  }
}

// omega'(:, b) = sum_{(r, a) in col b, r0 <= r < r1} ( B(r, b) E_r + Rv_r[a] V'_r ): the
// contribution of this shard's rows (the gradient is linear in omega, so shard partials add).
// Work items are (M-chunk, column) pairs, chunk-major: one pass over all columns touches only
// kOmChunk rows of E and V', so the ~m_v-fold reuse of each gathered column is served from L2
// (a full-height pass has a working set of ~2 time blocks of E and V', beyond L2).
template <int NJ>  // M-chunk = 128 * NJ rows, NJ per thread
__global__ void __launch_bounds__(128) omega_prime_kernel(int c0, int c1, int r0, int r1, int ldm, int m_v,
                                                          const int32_t* ptr, const int32_t* erow,
                                                          const int16_t* eslot, const double* A, const double* Rv,
                                                          const double* E, const double* Vp, const int32_t* corder,
                                                          unsigned long long* next, double* Om) {
  constexpr int kChunk = 128 * NJ;
  __shared__ int sr[64];
  __shared__ double sb[64], sv[64];
  __shared__ long long s_item;
  const long long ncols = c1 - c0;
  const int nch = (ldm + kChunk - 1) / kChunk;
  // Items are claimed from a global counter: column entry counts vary widely, and a static
  // grid-stride split lets blocks drift apart until the in-flight columns span most of the array
  // (no L2 reuse of the gathered E/V' segments).  Dynamic claiming keeps them a contiguous window.
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = static_cast<long long>(atomicAdd(next, 1ull));
    __syncthreads();
    const long long e = s_item;
    if (e >= ncols * nch) break;
    const int q = static_cast<int>(e / ncols);
    const int kc = static_cast<int>(e - static_cast<long long>(q) * ncols);
    const int b = corder ? corder[kc] : c0 + kc;
    const int jb = q * kChunk + threadIdx.x;
    const int p0 = ptr[b], p1 = ptr[b + 1];
    double acc[NJ];
#pragma unroll
    for (int u = 0; u < NJ; ++u) acc[u] = 0.0;
    for (int pb = p0; pb < p1; pb += 64) {
      __syncthreads();
      if (threadIdx.x < 64) {  // entries of other shards' rows get weight 0 (fixed summation order)
        const int p = pb + threadIdx.x;
        int r = r0;
        double bb = 0.0, vv = 0.0;
        if (p < p1) {
          const int rr = erow[p];
          if (rr >= r0 && rr < r1) {
            const int sl = eslot[p];
            r = rr;
            bb = sl < 0 ? 1.0 : -A[static_cast<size_t>(rr) * m_v + sl];
            vv = sl < 0 ? 0.0 : Rv[static_cast<size_t>(rr) * m_v + sl];
          }
        }
        sr[threadIdx.x] = r;
        sb[threadIdx.x] = bb;
        sv[threadIdx.x] = vv;
      }
      __syncthreads();
      const int cnt = min(64, p1 - pb);
#pragma unroll 2
      for (int t = 0; t < cnt; ++t) {
        const size_t o = static_cast<size_t>(sr[t]) * ldm;
        const double cb = sb[t], cv = sv[t];
#pragma unroll
        for (int u = 0; u < NJ; ++u) {
          const int j = jb + 128 * u;
          if (j < ldm) acc[u] = fma(cv, __ldg(&Vp[o + j]), fma(cb, __ldg(&E[o + j]), acc[u]));
        }
      }
    }
    double* out = Om + static_cast<size_t>(b) * ldm;
#pragma unroll
    for (int u = 0; u < NJ; ++u)
      if (jb + 128 * u < ldm) out[jb + 128 * u] = acc[u];
  }
}

static void launch_omega_prime(stgp_ctx* ctx, int c0, int c1, int r0, int r1, int ldm, int m_v, const int32_t* ptr,
                               const int32_t* erow, const int16_t* eslot, const double* A, const double* Rv,
                               const double* E, const double* Vp, const int32_t* corder, double* Om) {
  static const int nj_env = [] {
    const char* e = std::getenv("STGP_OM_NJ");  // tuning switch: 1, 2, 4 or 8 (rows per thread)
    return e ? std::atoi(e) : 2;
  }();
  const int nj = nj_env == 1 || nj_env == 2 || nj_env == 4 || nj_env == 8 ? nj_env : 2;
  const long long items = static_cast<long long>(c1 - c0) * ((ldm + 128 * nj - 1) / (128 * nj));
  const int grid = static_cast<int>(std::min<long long>(items, ctx->num_sms * 16));
  unsigned long long* next = claim_counter(ctx);
#define STGP_OM(NJ)                                                                                            \
  omega_prime_kernel<NJ><<<grid, 128, 0, ctx->stream>>>(c0, c1, r0, r1, ldm, m_v, ptr, erow, eslot, A, Rv, E, Vp, \
                                                        corder, next, Om)
  switch (nj) {
    case 1: STGP_OM(1); break;
    case 4: STGP_OM(4); break;
    case 8: STGP_OM(8); break;
    default: STGP_OM(2);
  }
#undef STGP_OM
  launched(ctx);
}

// min over rows [r0, r1) of the first (smallest) neighbour index, and r0 itself
__global__ void halo_kernel(int r0, int r1, int m_v, const int32_t* nbr, int* out) {
  int mn = r0;
  for (int i = r0 + blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += gridDim.x * blockDim.x) {
    const int j = nbr[static_cast<size_t>(i) * m_v];
    if (j >= 0 && j < mn) mn = j;
  }
  atomicMin(out, mn);
}

// sum_{j, i} Om(j, i) dk(z_j, p_i) over columns [c0, c1): per-block partials (6)
__global__ void __launch_bounds__(256) upair_grad_kernel(int c0, int c1, int M, int ldm, ZPts z, const double* x,
                                                         const double* y, const int32_t* tid, DevKernel k, double inv_c,
                                                         LagTable lt, const double* Om, double* part) {
  double g[6] = {0, 0, 0, 0, 0, 0};
  const MaternPoly mp = matern_poly(k.nu_code);
  for (int i = c0 + blockIdx.x; i < c1; i += gridDim.x) {
    const double xi = x[i], yi = y[i];
    const int ti = tid[i];
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
      const TF f = lt.get(z.ztid[j], ti);
      double kg[6];
      const double dx = z.zx[j] - xi, dy = z.zy[j] - yi;
      gneiting_grad_bf(k, mp, inv_c, fma(dx, dx, dy * dy), f, kg);
      const double wgt = Om[static_cast<size_t>(i) * ldm + j];
#pragma unroll
      for (int q = 0; q < 6; ++q) g[q] = fma(wgt, kg[q], g[q]);
    }
  }
  __shared__ double red[6][256];
#pragma unroll
  for (int q = 0; q < 6; ++q) red[q][threadIdx.x] = g[q];
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
#pragma unroll
      for (int q = 0; q < 6; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 6) part[static_cast<size_t>(blockIdx.x) * 6 + threadIdx.x] = red[threadIdx.x][0];
}

// Sigma_m pairs: sum_{j1 >= j2} w(j1, j2) dk(z_j1, z_j2), w = wsig(j1,j1) or wsig(j1,j2) + wsig(j2,j1)
__global__ void __launch_bounds__(256) sigma_pair_grad_kernel(int M, int ldm, ZPts z, DevKernel k, double inv_c,
                                                              LagTable lt, const double* Ws, double* part) {
  double g[6] = {0, 0, 0, 0, 0, 0};
  const MaternPoly mp = matern_poly(k.nu_code);
  const long long total = static_cast<long long>(M) * M;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int j1 = static_cast<int>(e / M), j2 = static_cast<int>(e % M);
    if (j2 > j1) continue;
    const double wgt = j1 == j2 ? Ws[static_cast<size_t>(j1) * ldm + j1]
                                : Ws[static_cast<size_t>(j2) * ldm + j1] + Ws[static_cast<size_t>(j1) * ldm + j2];
    const TF f = lt.get(z.ztid[j1], z.ztid[j2]);
    double kg[6];
    const double dx = z.zx[j1] - z.zx[j2], dy = z.zy[j1] - z.zy[j2];
    gneiting_grad_bf(k, mp, inv_c, fma(dx, dx, dy * dy), f, kg);
#pragma unroll
    for (int q = 0; q < 6; ++q) g[q] = fma(wgt, kg[q], g[q]);
  }
  __shared__ double red[6][256];
#pragma unroll
  for (int q = 0; q < 6; ++q) red[q][threadIdx.x] = g[q];
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
#pragma unroll
      for (int q = 0; q < 6; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 6) part[static_cast<size_t>(blockIdx.x) * 6 + threadIdx.x] = red[threadIdx.x][0];
}

// M x M helper: C = 0.5 * y y^T + S + 0.5 * (Kinv - I)   (lower+upper)
__global__ void wsig_assemble_kernel(int M, int ldm, const double* yhat, const double* S, const double* Kinv,
                                     double* out) {
  const long long total = static_cast<long long>(ldm) * ldm;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e % ldm), c = static_cast<int>(e / ldm);
    double v = 0.0;
    if (r < M && c < M) {
      // sym(S): S holds V' F^T, both triangles
      const double s = 0.5 * (S[static_cast<size_t>(c) * ldm + r] + S[static_cast<size_t>(r) * ldm + c]);
      v = 0.5 * yhat[r] * yhat[c] + s + 0.5 * (Kinv[e] - (r == c ? 1.0 : 0.0));
    }
    out[e] = v;
  }
}

__global__ void block_sum_kernel(const double* v, long long n, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void block_sumlog_kernel(const double* v, long long n, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    s += log(v[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// deterministic dot product partials
__global__ void dot_kernel(const double* a, const double* b, long long n, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    s = fma(a[i], b[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

}  // namespace

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
double dev_dot(stgp_ctx* ctx, const double* a, const double* b, long long n, Reducer& red) {
  const int blocks = grid_for(n, kT, 1024);
  red.ensure(blocks, 1);
  dot_kernel<<<blocks, kT, 0, ctx->stream>>>(a, b, n, red.part.get());
  launched(ctx);
  return red.finish(ctx, blocks, 1)[0];
}

// L2 schedule for the W-gathering kernels (rows kernels, V', E/F, omega'): row i reads the
// ~m_v columns W(:, N_i) of 7 KB each, and the rows sharing a column are its space-time
// neighbours.  Index order interleaves stations randomly within a time block, so those rows run
// thousands of rows apart and every column is re-fetched from HBM ~m_v times.  Processing rows
// by (time bucket of >= kBucketRows rows, Morton code of (x, y)) keeps the in-flight rows'
// neighbour columns (current and previous bucket, same spatial patch) L2-resident.  Only the
// processing order changes: per-row outputs are identical, block partial sums are regrouped.
std::vector<int32_t> locality_order(const stgp_dataset* ds, int lo, int hi) {
  constexpr int kBucketRows = 4096;
  std::vector<int32_t> out;
  if (hi <= lo) return out;
  const size_t nT = ds->Tdata.size();
  std::vector<int> cnt(nT, 0), bucket(nT, 0);
  for (int32_t t : ds->htid) ++cnt[static_cast<size_t>(t)];
  int b = 0, acc = 0;
  for (size_t t = 0; t < nT; ++t) {
    bucket[t] = b;
    acc += cnt[t];
    if (acc >= kBucketRows) {
      ++b;
      acc = 0;
    }
  }
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
  for (int i = 0; i < ds->n; ++i) {
    x0 = std::min(x0, ds->hx[i]);
    x1 = std::max(x1, ds->hx[i]);
    y0 = std::min(y0, ds->hy[i]);
    y1 = std::max(y1, ds->hy[i]);
  }
  const double sx = x1 > x0 ? 65535.0 / (x1 - x0) : 0.0, sy = y1 > y0 ? 65535.0 / (y1 - y0) : 0.0;
  auto spread = [](uint64_t v) {  // 16 bits -> even bit positions
    v &= 0xffff;
    v = (v | (v << 8)) & 0x00ff00ff;
    v = (v | (v << 4)) & 0x0f0f0f0f;
    v = (v | (v << 2)) & 0x33333333;
    v = (v | (v << 1)) & 0x55555555;
    return v;
  };
  std::vector<std::pair<uint64_t, int32_t>> key(static_cast<size_t>(hi - lo));
  for (int i = lo; i < hi; ++i) {
    const uint64_t qx = static_cast<uint64_t>((ds->hx[i] - x0) * sx), qy = static_cast<uint64_t>((ds->hy[i] - y0) * sy);
    const uint64_t bk = static_cast<uint64_t>(bucket[static_cast<size_t>(ds->htid[static_cast<size_t>(i)])]);
    key[static_cast<size_t>(i - lo)] = {(bk << 32) | spread(qx) | (spread(qy) << 1), i};
  }
  std::sort(key.begin(), key.end());
  out.resize(key.size());
  for (size_t k = 0; k < key.size(); ++k) out[k] = key[k].second;
  return out;
}

ZPts zpts(const stgp_structure* s) { return ZPts{s->lr.zx.get(), s->lr.zy.get(), s->lr.ztid.get()}; }

void lowrank_setup(stgp_structure* s, const stgp_inducing* ind) {
  if (s->m_v > kMaxGatherM) config_error("VIF: neighbour sets wider than 512 are not supported");
  LowRank& L = s->lr;
  L.M = ind->M();
  L.zxyt = ind->xyt;
  L.ldm = std::max(16, (L.M + 15) / 16 * 16);
  std::vector<double> zx(L.M), zy(L.M), zt(L.M);
  for (int j = 0; j < L.M; ++j) {
    zx[j] = ind->xyt[3 * j];
    zy[j] = ind->xyt[3 * j + 1];
    zt[j] = ind->xyt[3 * j + 2];
    if (!std::isfinite(zx[j]) || !std::isfinite(zy[j]) || !std::isfinite(zt[j]))
      data_error("SpaceTimePoint: coordinates and time must be finite");
  }
  // time groups: data times, then distinct inducing times
  std::set<double> it(zt.begin(), zt.end());
  std::vector<double> Ti(it.begin(), it.end());
  std::vector<int32_t> ztid(L.M);
  const int nD = static_cast<int>(s->ds->Tdata.size());
  for (int j = 0; j < L.M; ++j)
    ztid[j] = nD + static_cast<int>(std::lower_bound(Ti.begin(), Ti.end(), zt[j]) - Ti.begin());
  s->ti.T = s->ds->Tdata;
  s->ti.T.insert(s->ti.T.end(), Ti.begin(), Ti.end());
  s->ti.build();
  s->ti_dirty = true;
  compute_halo(s);
  cudaStream_t st = s->ds->ctx->stream;
  const char* om = std::getenv("STGP_ORDER");  // tuning switch: none | rows | all (default none)
  const std::string omode = om ? om : "none";
  s->order_rows = omode == "rows" || omode == "all";
  s->order_gather = omode == "all";
  if (s->kind == STGP_VIF && (s->order_rows || s->order_gather)) {
    const std::vector<int32_t> ro = locality_order(s->ds, s->row_begin, s->row_end);
    const std::vector<int32_t> co = locality_order(s->ds, s->col_begin, s->row_end);
    if (!ro.empty()) s->rorder.upload(ro.data(), ro.size(), st);
    if (!co.empty()) s->corder.upload(co.data(), co.size(), st);
  }
  L.zx.upload(zx.data(), L.M, st);
  L.zy.upload(zy.data(), L.M, st);
  L.zt.upload(zt.data(), L.M, st);
  L.ztid.upload(ztid.data(), L.M, st);
}

// Sigma_m Cholesky with the jitter ladder (inducing.cpp:250-261)
void build_basis(stgp_structure* s) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const DevKernel k = dev_kernel(s->th);
  const LagTable lt = lag_view(s->lt);
  const double jitter = 1e-8 * s->th.sigma1_2;
  L.Lm.ensure(static_cast<size_t>(L.ldm) * L.ldm);
  for (int attempt = 0; attempt < 2; ++attempt) {
    sigma_m_kernel<<<grid_for(static_cast<long long>(L.ldm) * L.ldm), kT, 0, ctx->stream>>>(
        zpts(s), L.M, L.ldm, k, lt, jitter, attempt == 0 ? 0.0 : 9.0 * jitter, L.Lm.get());
    launched(ctx);
    if (dev_cholesky(ctx, L.Lm.get(), L.ldm, L.ldm)) {
      L.logdet_m = dev_logdet_chol(ctx, L.Lm.get(), L.ldm, L.M);
      L.Lminv.ensure(static_cast<size_t>(L.ldm) * L.ldm);
      dev_tri_inverse(ctx, L.Lm.get(), L.ldm, L.ldm, L.Lminv.get());
      return;
    }
  }
  numeric_error("InducingBasis: inducing covariance is not positive definite");
}

// U (kept) and W = L_m^{-1} U for columns [c0, c1): explicit triangular inverse + TRMM
void build_cross(stgp_structure* s, int c0, int c1, bool /*keep_U*/) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const size_t total = static_cast<size_t>(L.ldm) * s->n;
  L.U.ensure(total);
  L.W.ensure(total);
  {
    ProfRegion pr(ctx, "U_cross_cov");
    const DevKernel k = dev_kernel(s->th);
    auto kern = k.nu_code == kNuGeneral ? cross_cov_kernel<true> : cross_cov_kernel<false>;
    kern<<<std::max(1, std::min(c1 - c0, ctx->num_sms * 16)), 128, 0, ctx->stream>>>(
        zpts(s), L.M, L.ldm, s->ds->x.get(), s->ds->y.get(), s->ds->tid.get(), c0, c1, k, lag_view(s->lt),
        L.U.get());
    launched(ctx);
  }
  ProfRegion pr(ctx, "W_trmm");
  lr_trmm(ctx, L.Lminv.get(), L.ldm, L.U.get() + static_cast<size_t>(c0) * L.ldm, c1 - c0, false,
          L.W.get() + static_cast<size_t>(c0) * L.ldm);
}

void compute_halo(stgp_structure* s) {
  stgp_ctx* ctx = s->ds->ctx;
  int init = s->row_begin;
  DevBuf<int>& d = ctx->iscr;
  d.ensure(1);
  d.upload(&init, 1, ctx->stream);
  if (s->row_end > s->row_begin && s->kind != STGP_FITC) {
    halo_kernel<<<grid_for(s->row_end - s->row_begin), kT, 0, ctx->stream>>>(s->row_begin, s->row_end, s->m_v,
                                                                            s->nbr.get(), d.get());
    launched(ctx);
  }
  d.download(&s->col_begin, 1, ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
}

void ensure_csc(stgp_structure* s) {
  if (s->csc_built) return;
  stgp_ctx* ctx = s->ds->ctx;
  const int n = s->n, m_v = s->m_v;
  DevBuf<int32_t> cnt(static_cast<size_t>(n) + 1), fillc(static_cast<size_t>(n));
  cnt.zero(ctx->stream);
  fillc.zero(ctx->stream);
  csc_count_kernel<<<grid_for(static_cast<long long>(n) * m_v), kT, 0, ctx->stream>>>(n, m_v, s->nbr.get(), cnt.get());
  launched(ctx);
  s->csc_ptr.ensure(static_cast<size_t>(n) + 1);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.get(), s->csc_ptr.get(), n + 1, ctx->stream);
  DevBuf<unsigned char> tmp(tmp_bytes);
  cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, cnt.get(), s->csc_ptr.get(), n + 1, ctx->stream);
  launched(ctx);
  int nnz = 0;
  STGP_CUDA(cudaMemcpyAsync(&nnz, s->csc_ptr.get() + n, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  s->csc_row.ensure(static_cast<size_t>(nnz));
  s->csc_slot.ensure(static_cast<size_t>(nnz));
  csc_fill_kernel<<<grid_for(static_cast<long long>(n) * (m_v + 1)), kT, 0, ctx->stream>>>(
      n, m_v, s->nbr.get(), s->csc_ptr.get(), fillc.get(), s->csc_row.get(), s->csc_slot.get());
  launched(ctx);
  csc_sort_kernel<<<grid_for(n), kT, 0, ctx->stream>>>(n, s->csc_ptr.get(), s->csc_row.get(), s->csc_slot.get());
  launched(ctx);
  s->csc_built = true;
}

void b_apply(stgp_structure* s, const double* v, double* out) {
  stgp_ctx* ctx = s->ds->ctx;
  b_apply_kernel<<<grid_for(s->n), kT, 0, ctx->stream>>>(0, s->n, s->m_v, s->nbr.get(), s->A.get(), v, out);
  launched(ctx);
}
void bt_apply(stgp_structure* s, const double* v, double* out) {
  stgp_ctx* ctx = s->ds->ctx;
  ensure_csc(s);
  bt_apply_kernel<<<grid_for(s->n), kT, 0, ctx->stream>>>(0, s->n, s->m_v, s->csc_ptr.get(), s->csc_row.get(),
                                                          s->csc_slot.get(), s->A.get(), v, out);
  launched(ctx);
}

void scale_cols(stgp_ctx* ctx, const double* in, int ldm, long long ncols, const double* sc, bool rsqrt_of, double* out) {
  scale_cols_kernel<<<grid_for(static_cast<long long>(ldm) * ncols), kT, 0, ctx->stream>>>(in, ldm, ncols, sc, rsqrt_of,
                                                                                          out);
  launched(ctx);
}
__global__ void add_identity_kernel(double* A, int ld) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += gridDim.x * blockDim.x)
    A[static_cast<size_t>(i) * ld + i] += 1.0;
}
void add_identity(stgp_ctx* ctx, double* A, int ld) {
  add_identity_kernel<<<grid_for(ld), kT, 0, ctx->stream>>>(A, ld);
  launched(ctx);
}
void vsub(stgp_ctx* ctx, long long n, const double* a, const double* b, double* out) {
  vsub_kernel<<<grid_for(n), kT, 0, ctx->stream>>>(n, a, b, out);
  launched(ctx);
}
void vadd(stgp_ctx* ctx, long long n, const double* a, const double* b, double* out) {
  vadd_kernel<<<grid_for(n), kT, 0, ctx->stream>>>(n, a, b, out);
  launched(ctx);
}
void set_identity(stgp_ctx* ctx, double* A, int ld) {
  set_identity_kernel<<<grid_for(static_cast<long long>(ld) * ld), kT, 0, ctx->stream>>>(A, ld, ld);
  launched(ctx);
}
void div_vec(stgp_ctx* ctx, int n, const double* x, const double* d, double* y) {
  div_kernel<<<grid_for(n), kT, 0, ctx->stream>>>(n, x, d, y);
  launched(ctx);
}
double dev_sum(stgp_ctx* ctx, const double* v, long long n, Reducer& red) {
  const int blocks = grid_for(n, kT, 1024);
  red.ensure(blocks, 1);
  block_sum_kernel<<<blocks, kT, 0, ctx->stream>>>(v, n, red.part.get());
  launched(ctx);
  return red.finish(ctx, blocks, 1)[0];
}
double dev_sum_log(stgp_ctx* ctx, const double* v, long long n, Reducer& red) {
  const int blocks = grid_for(n, kT, 1024);
  red.ensure(blocks, 1);
  block_sumlog_kernel<<<blocks, kT, 0, ctx->stream>>>(v, n, red.part.get());
  launched(ctx);
  return red.finish(ctx, blocks, 1)[0];
}
// Ws <- L_m^{-T} Ws L_m^{-1} with the basis' explicit inverse factor
void transform_wsig(stgp_ctx* ctx, const double* Lminv, int ldm, double* Ws) { dev_congruence_t(ctx, Lminv, ldm, ldm, Ws); }

void lr_trmm(stgp_ctx* ctx, const double* Lminv, int ldm, const double* B, long long ncols, bool transpose, double* C) {
  if (ozaki_for(ldm) && ozaki_trmm_enabled())
    ozaki_trmm_left(ctx, Lminv, ldm, ldm, B, ldm, ncols, transpose, C, ldm);
  else
    dev_trmm_left(ctx, Lminv, ldm, ldm, B, ldm, ncols, transpose, C, ldm);
}
std::vector<double> upair_grad(stgp_structure* s, const double* Om, int c0, int c1) {
  stgp_ctx* ctx = s->ds->ctx;
  const int ub = std::max(1, std::min(c1 - c0, ctx->num_sms * 8));
  Reducer r;
  r.ensure(ub, 6);
  upair_grad_kernel<<<ub, 256, 0, ctx->stream>>>(c0, c1, s->lr.M, s->lr.ldm, zpts(s), s->ds->x.get(), s->ds->y.get(),
                                                 s->ds->tid.get(), dev_kernel(s->th), 1.0 / s->th.c, lag_view(s->lt), Om,
                                                 r.part.get());
  launched(ctx);
  return r.finish(ctx, ub, 6);
}
std::vector<double> sigma_pair_grad(stgp_structure* s, const double* Ws) {
  stgp_ctx* ctx = s->ds->ctx;
  const int M = s->lr.M;
  const int sb = grid_for(static_cast<long long>(M) * M, 256, 1024);
  Reducer r;
  r.ensure(sb, 6);
  sigma_pair_grad_kernel<<<sb, 256, 0, ctx->stream>>>(M, s->lr.ldm, zpts(s), dev_kernel(s->th), 1.0 / s->th.c,
                                                      lag_view(s->lt), Ws, r.part.get());
  launched(ctx);
  return r.finish(ctx, sb, 6);
}

// ---------------------------------------------------------------------------
// builds
// ---------------------------------------------------------------------------
void vif_build(stgp_structure* s) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  prepare_tables(s);
  const double nug = s->policy == STGP_OBSERVATION ? s->th.sigma2 : 0.0;
  if (L.M == 0) {
    run_rows(s, kModeBuild, nullptr, 0, nug);
    s->built = true;
    return;
  }
  const int rb = s->row_begin, re = s->row_end, hb = s->col_begin, ldm = L.ldm;
  {
    ProfRegion pr(ctx, "basis");
    build_basis(s);
  }
  build_cross(s, hb, re, false);  // W for this shard's rows and their halo
  {
    RowArgs ra = row_args(s, L.W.get(), ldm, nug);
    if (s->m_v <= kKmax - 1 && s->policy == STGP_OBSERVATION) {
      L.Lfac.ensure(static_cast<size_t>(s->n) * lfac_stride_for(s->m_v));
      ra.Lfac_out = L.Lfac.get();
    }
    run_rows_args(s, kModeBuild, ra);
  }
  // V' = W B^T (own columns) and K = I + sum_shards V' D^{-1} V'^T
  const size_t total = static_cast<size_t>(ldm) * s->n;
  L.Vp.ensure(total);
  if (re > rb) {
    ProfRegion pr(ctx, "vprime");
    if (!tile_vprime(s, L.W.get(), s->A.get(), L.Vp.get())) {
    vprime_kernel<<<std::min(re - rb, ctx->num_sms * 16), 128, 0, ctx->stream>>>(
        L.W.get(), ldm, s->nbr.get(), s->m_v, s->A.get(), rb, re, s->order_gather ? s->rorder.get() : nullptr,
        claim_counter(ctx), L.Vp.get());
    launched(ctx);
    }
  }
  ProfRegion prk(ctx, "K_gemm_chol");
  L.work1.ensure(total);
  const size_t off = static_cast<size_t>(rb) * ldm;
  if (!ozaki_for(ldm)) scale_cols(ctx, L.Vp.get() + off, ldm, re - rb, s->D.get() + rb, true, L.work1.get() + off);
  L.Mc.ensure(static_cast<size_t>(ldm) * ldm);
  STGP_CUDA(cudaMemsetAsync(L.Mc.get(), 0, sizeof(double) * ldm * ldm, ctx->stream));
  // S S^T as GEMMs over the lower blocks of a partition (dense.cu dev_syrk_blocked)
  if (re > rb) {
    static const int kblocks = [] {
      const char* e = std::getenv("STGP_KBLOCKS");
      return e ? std::max(1, std::atoi(e)) : 4;  // 5/8 of the GEMM flops; measured best at M = 906
    }();
    if (ozaki_for(ldm))  // S S^T on the int8 tensor cores (exactly symmetric result)
      ozaki_syrk_keep(ctx, ldm, re - rb, L.Vp.get() + off, ldm, s->D.get() + rb, L.Mc.get(), ldm, s->uid);
    else
      dev_syrk_blocked(ctx, ldm, re - rb, 1.0, L.work1.get() + off, ldm, L.Mc.get(), ldm, kblocks);
  }
  allreduce_sum(ctx, L.Mc.get(), static_cast<size_t>(ldm) * ldm);
  add_identity(ctx, L.Mc.get(), ldm);
  L.Kfull.ensure(static_cast<size_t>(ldm) * ldm);
  STGP_CUDA(cudaMemcpyAsync(L.Kfull.get(), L.Mc.get(), sizeof(double) * ldm * ldm, cudaMemcpyDeviceToDevice,
                            ctx->stream));
  if (!dev_cholesky(ctx, L.Mc.get(), ldm, ldm)) numeric_error("build_vif: Woodbury core factorization failed");
  L.logdet_M = dev_logdet_chol(ctx, L.Mc.get(), ldm, ldm);  // = log|M_core| - log|Sigma_m|
  s->built = true;
}

// ---------------------------------------------------------------------------
// NLL (approximations.cpp:352-384)
// ---------------------------------------------------------------------------
// rows_sum: this shard's sum of log D + u^2 / D.  Leaves W ur (all shards) in vecM.
static double vif_nll_given_u(stgp_structure* s, double rows_sum) {
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int rb = s->row_begin, re = s->row_end, ldm = L.ldm;
  std::vector<double> parts{rows_sum};
  allreduce_host(ctx, parts);
  double quad_lr = 0.0, logdet_lr = 0.0;
  if (L.M > 0) {
    // W ur = V' D^{-1} u (own columns, then summed over shards);  quad -= (W ur)' K^{-1} (W ur)
    L.vecN.ensure(s->n);
    L.vecM.ensure(ldm);
    L.vecM2.ensure(ldm);
    STGP_CUDA(cudaMemsetAsync(L.vecM.get(), 0, sizeof(double) * ldm, ctx->stream));
    if (re > rb) {
      div_vec(ctx, re - rb, s->u.get() + rb, s->D.get() + rb, L.vecN.get() + rb);
      dev_gemv(ctx, false, ldm, re - rb, 1.0, L.Vp.get() + static_cast<size_t>(rb) * ldm, ldm, L.vecN.get() + rb, 0.0,
               L.vecM.get());
    }
    allreduce_sum(ctx, L.vecM.get(), ldm);
    STGP_CUDA(cudaMemcpyAsync(L.vecM2.get(), L.vecM.get(), sizeof(double) * ldm, cudaMemcpyDeviceToDevice, ctx->stream));
    dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, L.vecM2.get(), ldm, 1, false);  // L_K^{-1} (W ur)
    quad_lr = dev_dot(ctx, L.vecM2.get(), L.vecM2.get(), ldm, s->red);
    logdet_lr = L.logdet_M;
  }
  return 0.5 * (parts[0] - quad_lr + logdet_lr + nll_const(s->n));
}

double lowrank_nll(stgp_structure* s) {
  stgp_ctx* ctx = s->ds->ctx;
  if (s->kind == STGP_FITC) return fitc_nll(s);
  if (s->policy != STGP_OBSERVATION) {  // approximations.cpp:369-371: through the Laplace algebra
    laplace_release(s);
    const double v = latent_policy_nll_dev(s);
    laplace_release(s);
    return v;
  }
  const int blocks = std::max(1, std::min(ceil_div(s->n, 256), ctx->num_sms * 4));
  s->red.ensure(blocks, 1);
  s->u.ensure(s->n);
  launch_nll_stored(s, blocks, s->u.get());
  const double rows_sum = s->red.finish(ctx, blocks, 1)[0];
  return vif_nll_given_u(s, rows_sum);
}

// ---------------------------------------------------------------------------
// VIF gradient (approximations.cpp:573-744), whitened (file header)
// ---------------------------------------------------------------------------
static void vif_grad(stgp_structure* s, double* nll_out, double* grad) {
  if (s->policy != STGP_OBSERVATION)
    numeric_error("nll_grad: analytic gradient is defined for the observation-policy structure driven by the optimizer");
  stgp_ctx* ctx = s->ds->ctx;
  LowRank& L = s->lr;
  const int n = s->n, ldm = L.ldm, rb = s->row_begin, re = s->row_end, hb = s->col_begin;
  if (L.M == 0) {  // plain Vecchia gradient on the residual structure
    std::vector<double> tot = run_rows(s, kModeGrad, nullptr, 0, s->th.sigma2);
    allreduce_host(ctx, tot);
    if (nll_out) *nll_out = 0.5 * (tot[0] + nll_const(n));
    for (int q = 0; q < 7; ++q) grad[q] = tot[1 + q];
    return;
  }
  const size_t total = static_cast<size_t>(ldm) * n;
  const size_t mm = static_cast<size_t>(ldm) * ldm;
  const size_t own = static_cast<size_t>(rb) * ldm, halo = static_cast<size_t>(hb) * ldm;
  cudaStream_t st = ctx->stream;
  // u = B r, NLL rows part
  std::unique_ptr<ProfRegion> ph(new ProfRegion(ctx, "g_nll"));
  const int nb = std::max(1, std::min(ceil_div(n, 256), ctx->num_sms * 4));
  s->red.ensure(nb, 1);
  s->u.ensure(n);
  launch_nll_stored(s, nb, s->u.get());
  const double rows_sum = s->red.finish(ctx, nb, 1)[0];
  const double nll_val = vif_nll_given_u(s, rows_sum);  // leaves W ur (all shards) in L.vecM
  ph.reset(new ProfRegion(ctx, "g_t_z"));
  if (nll_out) *nll_out = nll_val;
  double *t = L.tmp("t", n), *z = L.tmp("z", n), *Bz = L.tmp("Bz", n), *c0 = L.tmp("c0", n),
         *Rv = L.tmp("Rv", static_cast<size_t>(n) * s->m_v), *yhat = L.tmp("yhat", ldm), *S = L.tmp("S", mm),
         *Ws = L.tmp("Ws", mm);
  // yhat = K^{-1} W ur, t = W^T yhat, z = r - t (halo + own columns), Bz (own rows)
  STGP_CUDA(cudaMemcpyAsync(yhat, L.vecM.get(), sizeof(double) * ldm, cudaMemcpyDeviceToDevice, st));
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, yhat, ldm, 1, false);
  dev_trsm_left(ctx, L.Mc.get(), ldm, ldm, yhat, ldm, 1, true);
  dev_gemv(ctx, true, ldm, re - hb, 1.0, L.W.get() + halo, ldm, yhat, 0.0, t + hb);
  axpby_kernel<<<grid_for(re - hb), kT, 0, st>>>(re - hb, 1.0, s->r.get() + hb, -1.0, t + hb, z + hb);
  launched(ctx);
  b_apply_kernel<<<grid_for(re - rb), kT, 0, st>>>(rb, re, s->m_v, s->nbr.get(), s->A.get(), z, Bz);
  launched(ctx);
  // K^{-1} (explicit, M x M) and X = K^{-1} V' (own columns) as one GEMM
  ph.reset(new ProfRegion(ctx, "g_X_gemm"));
  L.Kinv.ensure(mm);
  dev_chol_inverse(ctx, L.Mc.get(), ldm, ldm, L.Kinv.get());
  L.work1.ensure(total);
  if (re > rb) {
    if (ozaki_for(ldm))  // K^{-1} is symmetric: X_r = K^{-1} V'_r row by row on the int8 tensor cores
      ozaki_gemm_rows(ctx, re - rb, ldm, ldm, L.Vp.get() + own, ldm, L.Kinv.get(), ldm, L.work1.get() + own, ldm);
    else
      dev_gemm(ctx, false, false, ldm, re - rb, ldm, 1.0, L.Kinv.get(), ldm, L.Vp.get() + own, ldm, 0.0,
               L.work1.get() + own, ldm);
  }
  // per-row Phi_i: direct pass + c0, Rv (own rows)
  ph.reset();
  RowArgs a = row_args(s, L.W.get(), ldm, s->th.sigma2);
  a.X = L.work1.get();
  a.Vp = L.Vp.get();
  a.z = z;
  a.Bz = Bz;
  a.D_in = s->D.get();
  a.c0_out = c0;
  a.Rv_out = Rv;
  a.A_out = nullptr;
  a.D_out = nullptr;
  if (L.Lfac.get() && s->m_v <= kKmax - 1) {  // stored factors from the build at this theta
    a.Lfac_in = L.Lfac.get();
    a.A_in = s->A.get();
  }
  if (a.Lfac_in && re > rb) {  // Ga by the tiled SDDMM (falls back to the rows kernel's DMMA pass)
    ProfRegion pg(ctx, "g_ga");
    double* Ga = L.tmp("Ga", static_cast<size_t>(n) * 32);
    if (tile_ga(s, L.W.get(), L.work1.get(), Ga)) a.Ga_in = Ga;
  }
  std::vector<double> rows = run_rows_args(s, kModeVifGrad, a);
  // E (in place of X) and F (own rows)
  ph.reset(new ProfRegion(ctx, "g_ef"));
  L.work2.ensure(total);
  if (re > rb && !tile_ef(s, L.W.get(), Rv, c0, s->D.get(), L.Vp.get(), yhat, Bz, L.work1.get(), L.work2.get())) {
    ef_kernel<<<std::min(re - rb, ctx->num_sms * 16), 128, 0, st>>>(rb, re, ldm, s->m_v, s->nbr.get(), Rv, c0,
                                                                    s->D.get(), L.W.get(), L.Vp.get(), yhat, Bz,
                                                                    s->order_gather ? s->rorder.get() : nullptr, claim_counter(ctx), L.work1.get(), L.work2.get());
    launched(ctx);
  }
  ph.reset(new ProfRegion(ctx, "g_S_gemm"));
  // W Phi W^T = sym(V' F^T) summed over shards -> wsig' = 0.5 yhat yhat^T + sym(V'F^T) + 0.5 (K^{-1} - I)
  if (re > rb && ozaki_for(ldm)) {  // S(i, j) = sum_r V'(i, r) F(j, r), or its transpose (symmetrised below)
    // V' D^{-1/2} was sliced for K in the build: reuse its digits, slice only F D^{1/2}
    if (!ozaki_gemm_kept(ctx, ldm, re - rb, L.work2.get() + own, ldm, s->D.get() + rb, S, ldm, s->uid))
      ozaki_gemm_cols(ctx, ldm, re - rb, L.work2.get() + own, ldm, L.Vp.get() + own, ldm, S, ldm);
  }
  else if (re > rb)
    dev_gemm(ctx, false, true, ldm, ldm, re - rb, 1.0, L.Vp.get() + own, ldm, L.work2.get() + own, ldm, 0.0, S, ldm);
  else
    STGP_CUDA(cudaMemsetAsync(S, 0, sizeof(double) * mm, st));
  allreduce_sum(ctx, S, mm);
  ph.reset(new ProfRegion(ctx, "g_wsig"));
  wsig_assemble_kernel<<<grid_for(static_cast<long long>(mm)), kT, 0, st>>>(L.M, ldm, yhat, S, L.Kinv.get(), Ws);
  launched(ctx);
  transform_wsig(ctx, L.Lminv.get(), ldm, Ws);
  // omega' over the columns this shard's rows touch, omega = L_m^{-T} omega'
  ph.reset(new ProfRegion(ctx, "g_omega"));
  ensure_csc(s);
  if (re > hb) {
    launch_omega_prime(ctx, hb, re, rb, re, ldm, s->m_v, s->csc_ptr.get(), s->csc_row.get(), s->csc_slot.get(),
                       s->A.get(), Rv, L.work1.get(), L.Vp.get(), s->order_gather ? s->corder.get() : nullptr,
                       L.work2.get());
    ph.reset(new ProfRegion(ctx, "g_omega_trmm"));
    L.work3.ensure(total);
    lr_trmm(ctx, L.Lminv.get(), ldm, L.work2.get() + halo, re - hb, true, L.work3.get() + halo);
  }
  // U-pair (this shard's omega) and Sigma_m-pair (rank 0) kernel gradients, then one all-reduce
  std::vector<double> g(7, 0.0);
  for (int qd = 0; qd < 7; ++qd) g[qd] = rows[1 + qd];
  ph.reset(new ProfRegion(ctx, "g_upair_sigma"));
  if (re > hb) {
    std::vector<double> gu = upair_grad(s, L.work3.get(), hb, re);
    for (int qd = 0; qd < 6; ++qd) g[1 + qd] += gu[qd];
  }
  if (ctx->rank == 0) {
    std::vector<double> gs = sigma_pair_grad(s, Ws);
    for (int qd = 0; qd < 6; ++qd) g[1 + qd] += gs[qd];
  }
  ph.reset();
  allreduce_host(ctx, g);
  for (int qd = 0; qd < 7; ++qd) grad[qd] = g[qd];
}

void lowrank_nll_grad(stgp_structure* s, double* nll, double* grad) {
  require_analytic_grad(s->th);
  if (s->kind == STGP_FITC) {
    fitc_nll_grad(s, nll, grad);
    return;
  }
  vif_grad(s, nll, grad);
}

}  // namespace stgp

extern "C" {
int stgp_inducing_create(stgp_ctx* ctx, int M, const double* xyt, stgp_inducing** out) {
  if (!ctx || !out || M < 0 || (M > 0 && !xyt)) {
    stgp::g_last_error = "stgp_inducing_create: bad argument";
    return STGP_ERR_CONFIG;
  }
  for (int i = 0; i < 3 * M; ++i)
    if (!std::isfinite(xyt[i])) {
      stgp::g_last_error = "SpaceTimePoint: coordinates and time must be finite";
      return STGP_ERR_DATA;
    }
  auto* ind = new stgp_inducing();
  ind->ctx = ctx;
  ind->xyt.assign(xyt, xyt + 3 * static_cast<size_t>(M));
  *out = ind;
  return STGP_OK;
}
int stgp_inducing_size(const stgp_inducing* ind, int* M, int* m_s, int* m_t) {
  if (!ind) return STGP_ERR_CONFIG;
  if (M) *M = ind->M();
  if (m_s) *m_s = ind->m_s;
  if (m_t) *m_t = ind->m_t;
  return STGP_OK;
}
int stgp_inducing_download(const stgp_inducing* ind, double* xyt) {
  if (!ind) return STGP_ERR_CONFIG;
  std::copy(ind->xyt.begin(), ind->xyt.end(), xyt);
  return STGP_OK;
}
void stgp_inducing_destroy(stgp_inducing* ind) { delete ind; }
}

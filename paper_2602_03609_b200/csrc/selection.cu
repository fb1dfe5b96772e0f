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
#include <chrono>
#include <cmath>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <set>
#include <type_traits>

#include <cub/device/device_radix_sort.cuh>
#include <cuda_fp16.h>

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
    double v = gneiting_eval<true>(k, spatial_dist(zx[a], zy[a], zx[b], zy[b]), f);
    if (r == c) {
      v = __dadd_rn(v, jit1);
      if (jit2 != 0.0) v = __dadd_rn(v, jit2);
    }
    A[e] = v;
  }
}


constexpr int kWB = 64;      // rows per block and columns per CTA
constexpr int kWKC = 16;     // K chunk of the off-diagonal update
constexpr int kWKS = 20;     // smem row stride (doubles): conflict-free DMMA fragment loads
constexpr int kWStages = 3;
constexpr int kWthreads = 256;
constexpr size_t kWStageDoubles = 2 * kWB * kWKS;
constexpr size_t kWsmem = sizeof(double) * (kWStages * kWStageDoubles + 64 * 65 + 2 * 64 + 2 * 64) + sizeof(int) * 64;
static_assert(kWStages * kWStageDoubles >= 64 * 65, "output tile aliases the staging ring");

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

// Blocked left-looking Cholesky in the oracle's order (chol_seq): every entry's chain
//   s = A[r][j]; for k < j: s = fma(-L[r][k], L[j][k], s)   (diagonal: r = j, then sqrt)
// is split at the panel start j0: the prefix k < j0 runs on the FP64 tensor pipe (DMMA = the
// sequential fma chain, scripts/exp/dmma_order.cu) for all rows below the panel in parallel, the
// rest k in [j0, j) inside the panel (<= 31 steps).  Row-major A, L (M x M).
constexpr int kCP = 32;  // panel width

// rows [j0, M) x panel columns [j0, j0 + pw): running values A[r][j] - sum_{k<j0} L[r][k] L[j][k]
__global__ void __launch_bounds__(128) chol_panel_update_kernel(const double* A, int M, int j0, int pw, double* L) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, grp = lane >> 2, tig = lane & 3;
  const int R0 = j0 + blockIdx.x * 64 + 16 * w;
  double acc[2][4][2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = R0 + 8 * u + grp, j = j0 + 8 * v + 2 * tig + h;
        acc[u][v][h] = (r < M && j < j0 + pw) ? A[static_cast<size_t>(r) * M + j] : 0.0;
      }
  const double* ra[2];
  const double* rb[4];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int r = R0 + 8 * u + grp;
    ra[u] = r < M ? L + static_cast<size_t>(r) * M + tig : nullptr;
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int j = j0 + 8 * v + grp;
    rb[v] = j < j0 + pw ? L + static_cast<size_t>(j) * M + tig : nullptr;
  }
  for (int kb = 0; kb < j0; kb += 4) {
    double fa[2], fb[4];
#pragma unroll
    for (int u = 0; u < 2; ++u) fa[u] = ra[u] ? -ra[u][kb] : 0.0;
#pragma unroll
    for (int v = 0; v < 4; ++v) fb[v] = rb[v] ? rb[v][kb] : 0.0;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) dmma_f64(acc[u][v][0], acc[u][v][1], fa[u], fb[v]);
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = R0 + 8 * u + grp, j = j0 + 8 * v + 2 * tig + h;
        if (r < M && j < j0 + pw) L[static_cast<size_t>(r) * M + j] = acc[u][v][h];
      }
}

// the panel's in-panel chain: column by column, the diagonal (thread of row j), then every row
// below; one CTA, rows strided over the threads
__global__ void __launch_bounds__(1024) chol_panel_factor_kernel(int M, int j0, int pw, double* L, int* fail) {
  __shared__ double sP[kCP][kCP + 1];  // the panel's diagonal block (rows j0.., cols j0..)
  __shared__ double s_d;
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int jj = 0; jj < pw; ++jj) {
    const int j = j0 + jj;
    if (threadIdx.x == 0) {
      double acc = L[static_cast<size_t>(j) * M + j];
      for (int k = 0; k < jj; ++k) acc = __fma_rn(-sP[jj][k], sP[jj][k], acc);
      if (acc <= 0.0) s_bad = 1;
      const double d = __dsqrt_rn(acc);
      s_d = d;
      sP[jj][jj] = d;
      L[static_cast<size_t>(j) * M + j] = d;
    }
    __syncthreads();
    if (s_bad) break;
    const double d = s_d;
    for (int r = j + 1 + threadIdx.x; r < M; r += blockDim.x) {
      const double* Lr = L + static_cast<size_t>(r) * M + j0;
      double sv = Lr[jj];
      for (int k = 0; k < jj; ++k) sv = __fma_rn(-Lr[k], sP[jj][k], sv);
      const double v = __ddiv_rn(sv, d);
      L[static_cast<size_t>(r) * M + j] = v;
      if (r - j0 < kCP) sP[r - j0][jj] = v;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && s_bad) *fail = 1;
}

// Zero-padded copy of L with a 16-double row stride (cp.async alignment).
__global__ void pad_rows_kernel(const double* L, int M, int ldL, double* Lp) {
  const long long total = static_cast<long long>(M) * ldL;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / ldL), c = static_cast<int>(e % ldL);
    Lp[e] = c < M ? L[static_cast<size_t>(r) * M + c] : 0.0;
  }
}

// W(:, i) = L^{-1} k_m(p_i) for 64 columns per CTA, row blocks of 64.  Every accumulator starts at
// k(z_r, p_i) and receives -L[r][c] w_c for c = 0, 1, ... in order -- the oracle's fwd_seq chain:
// the off-diagonal part c < r0 runs on the FP64 tensor pipe (mma.m8n8k4.f64 = the sequential fma
// chain over its k, scripts/exp/dmma_order.cu) over cp.async-staged 16-wide chunks in increasing c;
// the diagonal block is a column wavefront.  Warp w owns rows 16 (w/2).., columns 32 (w%2)...
template <bool GEN>
__global__ void __launch_bounds__(kWthreads) whiten_seq_kernel(const double* zx, const double* zy, const int32_t* ztid,
                                                              int M, int ldm, const double* x, const double* y,
                                                              const int32_t* tid, int col0, int n, DevKernel k,
                                                              LagTable lt, const double* Lp, int ldL, double* W) {
  extern __shared__ double sm[];
  __shared__ double sRcp[64];                         // rounded reciprocals of the diagonal block's pivots
  double* ring = sm;                                  // kWStages x [L 64 x kWKS | W 64 x kWKS]
  double* sOut = sm;                                  // [64 cols][65] (aliases the ring)
  double* sD = sm + kWStages * kWStageDoubles;        // [64][65]
  double* wrow = sD + 64 * 65;                        // [2][64]; [8] per warp in the diagonal solve
  double* sx = wrow + 2 * 64;                         // [64]
  double* sy = sx + 64;                               // [64]
  int* st = reinterpret_cast<int*>(sy + 64);
  const int i0 = col0 + blockIdx.x * kWB;  // columns [col0, n), 64 per block
  const int nc = min(kWB, n - i0);
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int grp = lane >> 2, tig = lane & 3, wr = wid >> 1, wc = wid & 1;
  if (t < kWB) {
    const int i = i0 + (t < nc ? t : 0);
    sx[t] = x[i];
    sy[t] = y[i];
    st[t] = tid[i];
  }
  __syncthreads();
  constexpr int kPieces = 2 * kWB * (kWKC / 2);
  static_assert(kPieces % kWthreads == 0, "staging split");
  for (int r0 = 0; r0 < M; r0 += kWB) {
    const int rb = min(kWB, M - r0);
    double acc[2][4][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + 16 * wr + 8 * u + grp, c = 32 * wc + 8 * v + 2 * tig + h;
          double val = 0.0;
          if (r < M && c < nc) {
            double pe, pb;
            lt.get2(ztid[r], st[c], pe, pb);
            TF f;
            f.pow_mE = pe;
            f.pow_mbh = pb;
            val = gneiting_eval<GEN>(k, spatial_dist(zx[r], zy[r], sx[c], sy[c]), f);  // k(z_r, p_i)
          }
          acc[u][v][h] = val;
        }
    const int nch = r0 / kWKC;
    if (nch > 0) {
      // per-thread source rows and shared offsets, fixed over the chunks of this row block
      const double* gsrc[kPieces / kWthreads];
      int soff[kPieces / kWthreads];
#pragma unroll
      for (int it = 0; it < kPieces / kWthreads; ++it) {
        const int pc = t + it * kWthreads;
        const int which = pc / (kWB * (kWKC / 2));  // 0: L rows, 1: W columns
        const int rem = pc % (kWB * (kWKC / 2));
        const int rr = rem / (kWKC / 2), piece = rem % (kWKC / 2);
        soff[it] = (which ? kWB * kWKS : 0) + rr * kWKS + 2 * piece;
        gsrc[it] = which == 0 ? Lp + static_cast<size_t>(min(r0 + rr, M - 1)) * ldL + 2 * piece
                              : W + static_cast<size_t>(i0 + (rr < nc ? rr : 0)) * ldm + 2 * piece;
      }
      auto stage = [&](int ch) {
        double* base = ring + static_cast<size_t>(ch % kWStages) * kWStageDoubles;
#pragma unroll
        for (int it = 0; it < kPieces / kWthreads; ++it) cp_async16(base + soff[it], gsrc[it] + ch * kWKC);
      };
#pragma unroll
      for (int ch = 0; ch < kWStages - 1; ++ch) {
        if (ch < nch) stage(ch);
        cp_async_commit();
      }
      for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait<kWStages - 2>();
        __syncthreads();
        if (ch + kWStages - 1 < nch) stage(ch + kWStages - 1);
        cp_async_commit();
        const double* sL = ring + static_cast<size_t>(ch % kWStages) * kWStageDoubles;
        const double* sW = sL + kWB * kWKS;
#pragma unroll
        for (int kb = 0; kb < kWKC; kb += 4) {
          double fa[2], fb[4];
#pragma unroll
          for (int u = 0; u < 2; ++u) fa[u] = -sL[(16 * wr + 8 * u + grp) * kWKS + kb + tig];
#pragma unroll
          for (int v = 0; v < 4; ++v) fb[v] = sW[(32 * wc + 8 * v + grp) * kWKS + kb + tig];
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) dmma_f64(acc[u][v][0], acc[u][v][1], fa[u], fb[v]);
        }
      }
      cp_async_wait<0>();
    }
    __syncthreads();
    // accumulators -> sOut (column-major: sOut[c][r]) and the diagonal block of L -> sD
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          sOut[(32 * wc + 8 * v + 2 * tig + h) * 65 + 16 * wr + 8 * u + grp] = acc[u][v][h];
    for (int e = t; e < 64 * 64; e += kWthreads) {
      const int rr = e / 64, cc = e % 64;
      sD[rr * 65 + cc] = (rr < rb && cc <= rr) ? Lp[static_cast<size_t>(r0 + rr) * ldL + r0 + cc] : 0.0;
    }
    if (t < rb) sRcp[t] = __drcp_rn(Lp[static_cast<size_t>(r0 + t) * ldL + r0 + t]);  // RN(1 / L_rr)
    __syncthreads();
    // diagonal block: the columns are independent forward substitutions, so warp w solves columns
    // 8w..8w+7 alone (lanes hold rows lane, lane + 32; lanes 0..7 divide, one column each): no
    // block-wide barrier per step.  Row r still receives -L[r][c] w_c for c = r0.. in order.
    {
      const int cb = 8 * wid;
      double* xw = wrow + 8 * wid;       // [8] per warp: row cl's values
      double* xq = wrow + 64 + 8 * wid;  // [8] per warp: their quotients
      double a0[8], a1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        a0[q] = sOut[(cb + q) * 65 + lane];
        a1[q] = sOut[(cb + q) * 65 + lane + 32];
      }
      // rows cl < 32 live in a0 (lanes), rows 32.. in a1: two loops without per-step selects, and
      // the second skips the a0 updates (all predicated off there)
      auto step = [&](const int cl, auto hi_t) {
        constexpr bool hi = decltype(hi_t)::value;
        const int own = cl & 31;
        // row cl's 8 values reach lanes 0..7 through the warp's shared slot (4 vector stores and
        // one load instead of 8 shuffles and 8 selects)
        if (lane == own) {
#pragma unroll
          for (int q = 0; q < 8; q += 2)
            reinterpret_cast<double2*>(xw)[q / 2] = hi ? make_double2(a1[q], a1[q + 1]) : make_double2(a0[q], a0[q + 1]);
        }
        __syncwarp();
        if (lane < 8) {  // lane q divides column cb + q's row cl and writes the result in place
          // x / L_cc correctly rounded from the rounded reciprocal y: q0 = RN(x y) is within an ulp
          // of x / L, r = x - q0 L is exact (fma), and RN(q0 + r y) = RN(x / L) (Markstein); r = 0
          // means q0 is the exact quotient (and keeps the sign of a zero x).  Bit-identical to
          // __ddiv_rn at a quarter of its latency on the wavefront's critical path.
          const double x = xw[lane], d = sD[cl * 65 + cl], y = sRcp[cl];
          const double q0 = __dmul_rn(x, y);
          const double r = __fma_rn(-q0, d, x);
          const double w = r == 0.0 ? q0 : __fma_rn(r, y, q0);
          xq[lane] = w;
          sOut[(cb + lane) * 65 + cl] = w;
        }
        __syncwarp();
        double wqv[8];
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          const double2 v2 = reinterpret_cast<const double2*>(xq)[q / 2];
          wqv[q] = v2.x;
          wqv[q + 1] = v2.y;
        }
        const double l0 = lane > cl ? -sD[lane * 65 + cl] : 0.0;
        const double l1 = lane + 32 > cl && lane + 32 < rb ? -sD[(lane + 32) * 65 + cl] : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double wv = wqv[q];
          if (!hi && lane > cl) a0[q] = __fma_rn(l0, wv, a0[q]);
          if (lane + 32 > cl) a1[q] = __fma_rn(l1, wv, a1[q]);
        }
      };
      const int rlo = min(rb, 32);
      for (int cl = 0; cl < rlo; ++cl) step(cl, std::false_type{});
      for (int cl = 32; cl < rb; ++cl) step(cl, std::true_type{});
    }
    __syncthreads();
    for (int e = t; e < 64 * 64; e += kWthreads) {  // coalesced column segments
      const int c = e / 64, rr = e % 64;
      if (c < nc && rr < rb) W[static_cast<size_t>(i0 + c) * ldm + r0 + rr] = sOut[c * 65 + rr];
    }
    __syncthreads();
  }
}

// r_i = sigma1_2 - |w_i|^2 (sequential fma from 0); degenerate flag.  One thread per row keeps
// the chain; the warp stages its 32 rows' k-chunks through shared memory with coalesced loads
// (a thread streaming its own 7 KB column alone touches 32 lines per warp load).
constexpr int kResRows = 128;
__global__ void __launch_bounds__(kResRows) resid_kernel(const double* W, int M, int ldm, int n, double s1,
                                                         double* resid, int* degen, double* wnorm) {
  __shared__ double sw[kResRows / 32][32][33];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  for (int base = blockIdx.x * kResRows; base < n; base += gridDim.x * kResRows) {
    const int i = base + threadIdx.x;
    const int r0 = base + wq * 32;
    double acc = 0.0;
    for (int k0 = 0; k0 < M; k0 += 32) {
      __syncwarp();
      for (int rr = 0; rr < 32; ++rr) {
        const int row = r0 + rr;
        sw[wq][rr][lane] = (row < n && k0 + lane < M) ? W[static_cast<size_t>(row) * ldm + k0 + lane] : 0.0;
      }
      __syncwarp();
      const int kn = min(32, M - k0);
      for (int kk = 0; kk < kn; ++kk) {
        const double v = sw[wq][lane][kk];
        acc = __fma_rn(v, v, acc);
      }
    }
    if (i < n) {
      const double r = M > 0 ? __dsub_rn(s1, acc) : s1;
      resid[i] = r;
      degen[i] = r <= 1e-7 * s1 ? 1 : 0;
      wnorm[i] = sqrt(acc) * (1.0 + 1e-12);  // >= |w_i| (the chain's rounding is ~M ulp)
    }
  }
}

// Half-precision copy of W for the d_r filter Gram: W16[i][k] = fp16(2^8 W[k][i]) (column i
// contiguous, ld16 a multiple of 64, zero padded).  The 2^8 scale keeps |w| >= 2^-22 normal.
constexpr double kW16Scale = 256.0;
__global__ void w16_kernel(const double* W, int M, int ldm, int n, int ld16, __half* W16) {
  const long long total = static_cast<long long>(n) * ld16;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = e / ld16;
    const int k = static_cast<int>(e - i * ld16);
    W16[e] = __double2half(k < M ? W[i * ldm + k] * kW16Scale : 0.0);
  }
}

// Spatial tiles of the d_r search: tile t holds rows sp[tile_off[t] .. tile_off[t+1]) (<= 64, one
// time bucket, Morton order).  Per tile: time-id range, bounding box, max |w| and min r over
// non-degenerate rows, degenerate flag, row-index range.
struct DrTiles {
  const int32_t *sp, *off, *bucket, *b_tile0, *b_tmax;
  const uint32_t* key;  // Morton key of the tile's first row (nondecreasing within a bucket)
  int *tmin, *tmax, *hasdeg, *imin, *imax;
  double *bx0, *bx1, *by0, *by1, *wmax, *rmin;
  // block-norm bound of the low-rank term: inducing points are split into G groups (inducing time x
  // spatial cell); A[t * G + g] = max over the tile's non-degenerate rows of |w_i[g]| / sqrt(r_i),
  // so |w_i . w_j| / sqrt(r_i r_j) <= sum_g A_Q[g] A_C[g].  Apre / rpre: prefix (buckets <= b) max / min.
  int G;
  double *A, *Apre, *rpre;
};

// (bucket << 32 | Morton(x, y)) sort keys and the identity permutation of the spatial tiles; bstart
// holds the nbucket + 1 bucket starts (the Morton part is 0 for unsorted data: index order)
__device__ __forceinline__ uint32_t spread16(uint32_t v) {
  v &= 0xffff;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__global__ void tile_keys_kernel(int n, const double* x, const double* y, const int* bstart, int nbucket, bool morton,
                                 double x0, double y0, double sx, double sy, uint64_t* keys, int32_t* iota) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int lo = 0, hi = nbucket;  // bucket b with bstart[b] <= i < bstart[b + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (bstart[mid] <= i) lo = mid; else hi = mid;
    }
    const uint32_t mk = morton ? (spread16(static_cast<uint32_t>((x[i] - x0) * sx)) |
                                  (spread16(static_cast<uint32_t>((y[i] - y0) * sy)) << 1))
                               : 0u;
    keys[i] = (static_cast<uint64_t>(lo) << 32) | mk;
    iota[i] = i;
  }
}

__global__ void tile_stats_kernel(DrTiles T, const double* x, const double* y, const double* resid,
                                  const int32_t* degen, const int32_t* tid, double s1) {
  const int tile = blockIdx.x;
  const int p0 = T.off[tile], p1 = T.off[tile + 1];
  __shared__ double sw[64], sr[64], sx0[64], sx1[64], sy0[64], sy1[64];
  __shared__ int smn[64], smx[64], sdg[64], sim[64], six[64];
  const int t = threadIdx.x;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double w = 0.0, r = inf, x0 = inf, x1 = -inf, y0 = inf, y1 = -inf;
  int mn = INT_MAX, mx = -1, dg = 0, im = INT_MAX, ix = -1;
  if (p0 + t < p1) {
    const int i = T.sp[p0 + t];
    mn = mx = tid[i];
    im = ix = i;
    x0 = x1 = x[i];
    y0 = y1 = y[i];
    if (degen[i]) {
      dg = 1;
    } else {
      r = resid[i];
      w = s1 - resid[i];
    }
  }
  sw[t] = w; sr[t] = r; sx0[t] = x0; sx1[t] = x1; sy0[t] = y0; sy1[t] = y1;
  smn[t] = mn; smx[t] = mx; sdg[t] = dg; sim[t] = im; six[t] = ix;
  __syncthreads();
  for (int o = 32; o > 0; o >>= 1) {
    if (t < o) {
      sw[t] = fmax(sw[t], sw[t + o]);
      sr[t] = fmin(sr[t], sr[t + o]);
      sx0[t] = fmin(sx0[t], sx0[t + o]);
      sx1[t] = fmax(sx1[t], sx1[t + o]);
      sy0[t] = fmin(sy0[t], sy0[t + o]);
      sy1[t] = fmax(sy1[t], sy1[t + o]);
      smn[t] = min(smn[t], smn[t + o]);
      smx[t] = max(smx[t], smx[t + o]);
      sdg[t] = sdg[t] | sdg[t + o];
      sim[t] = min(sim[t], sim[t + o]);
      six[t] = max(six[t], six[t + o]);
    }
    __syncthreads();
  }
  if (t == 0) {
    // |w|^2 = s1 - r up to one rounding of s1 (bounded by the 1e-11 factor of the prune test)
    T.wmax[tile] = sqrt(fmax(sw[0], 0.0) + 1e-15 * s1);
    T.rmin[tile] = sr[0];
    T.tmin[tile] = smn[0];
    T.tmax[tile] = smx[0];
    T.hasdeg[tile] = sdg[0];
    T.bx0[tile] = sx0[0];
    T.bx1[tile] = sx1[0];
    T.by0[tile] = sy0[0];
    T.by1[tile] = sy1[0];
    T.imin[tile] = sim[0];
    T.imax[tile] = six[0];
  }
}

constexpr int kMaxGroups = 48;

// A[tile][g] (see DrTiles): warp per row, lanes over k, group sums of squares in shared memory.
__global__ void __launch_bounds__(256) tile_groups_kernel(DrTiles T, const double* W, int ldm, int M,
                                                          const int32_t* kgroup, const double* resid,
                                                          const int32_t* degen) {
  __shared__ double sN[8][kMaxGroups], sA[8][kMaxGroups];
  const int tile = blockIdx.x, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = T.off[tile], p1 = T.off[tile + 1], G = T.G;
  for (int g = lane; g < G; g += 32) sA[w][g] = 0.0;
  for (int q = p0 + w; q < p1; q += 8) {
    const int i = T.sp[q];
    for (int g = lane; g < G; g += 32) sN[w][g] = 0.0;
    __syncwarp();
    const double* col = W + static_cast<size_t>(i) * ldm;
    for (int k = lane; k < M; k += 32) {
      const double v = col[k];
      atomicAdd(&sN[w][kgroup[k]], v * v);
    }
    __syncwarp();
    if (!degen[i]) {
      const double inv = 1.0 / sqrt(resid[i]);
      for (int g = lane; g < G; g += 32) sA[w][g] = fmax(sA[w][g], sqrt(sN[w][g]) * inv * (1.0 + 1e-12));
    }
    __syncwarp();
  }
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    double m = 0.0;
    for (int w2 = 0; w2 < 8; ++w2) m = fmax(m, sA[w2][g]);
    T.A[static_cast<size_t>(tile) * G + g] = m;
  }
}

constexpr int kQT = 64;   // queries per CTA
constexpr int kCT = 64;   // candidates per tile
constexpr int kKC = 16;   // K chunk staged per pipeline stage
constexpr int kKS = kKC + 4;  // smem row stride (doubles, = 4 mod 16): conflict-free DMMA fragment loads
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
  DrTiles T;
  // certified half-precision filter (0 = off): W16 (ld16 halves per column), |w_i| bounds
  const __half* W16;
  int ld16;
  const double* wnorm;
  int prune;                  // exact tile pruning (time-sorted rows)
  int tile0;                  // first query tile of this launch (rank shard)
  double s1;
  unsigned long long* stats;  // optional: [0] candidate tiles evaluated, [1] tiles pruned
};

// Upper bound of |rho_r| over the pairs of query tile Q and candidate tile C:
//   |k - w_i.w_j| / sqrt(r_i r_j) <= s1 T(u_min)^-E Matern(c h_min T(u_max)^-beta/2) / sqrt(rmin_Q rmin_C)
//                                    + sum_g A_Q[g] A_C[g]
// (T(u) and Matern are decreasing; h_min = box-to-box distance; degenerate rows excluded: they sit
// at d = 1).
// The (query tile, candidate tile) pieces of the bound: the temporal factors at the smallest lag
// (pe_min) and at the largest (pb_max), and the block bound wt of |w_i . w_j| / sqrt(r_i r_j).
__device__ __forceinline__ void tile_pair_terms(const DrArgs& a, int tminQ, int tmaxQ, const double* AQ, int ct,
                                                double& pe_min, double& pb_max, double& wt) {
  const DrTiles& T = a.T;
  // lags: C's times precede or equal Q's (time-sorted rows, j < i)
  const int tc0 = T.tmin[ct], tc1 = T.tmax[ct];
  double pb_dummy, pe_dummy;
  if (tc1 >= tminQ) {  // time ranges touch: u_min = 0
    pe_min = 1.0;
  } else {
    a.lt.get2(tminQ, tc1, pe_min, pb_dummy);
  }
  a.lt.get2(tmaxQ, tc0, pe_dummy, pb_max);
  wt = 0.0;
  const double* AC = T.A + static_cast<size_t>(ct) * T.G;
  for (int g = 0; g < T.G; ++g) wt += AQ[g] * AC[g];
}

__device__ __forceinline__ double tile_cmax(const DrArgs& a, double qx0, double qx1, double qy0, double qy1,
                                            double rQ, int ct, double pe_min, double pb_max, double wt) {
  const DrTiles& T = a.T;
  double mat = 1.0;
  if (a.k.nu_code != kNuGeneral) {  // general nu: the bound 1 (correlations are <= 1)
    const double dx = fmax(0.0, fmax(T.bx0[ct] - qx1, qx0 - T.bx1[ct]));
    const double dy = fmax(0.0, fmax(T.by0[ct] - qy1, qy0 - T.by1[ct]));
    const double hmin = sqrt(dx * dx + dy * dy) * (1.0 - 1e-12);
    const double xm = a.k.c * hmin * pb_max * (1.0 - 1e-12);
    mat = matern_from_exp(xm, exp(-xm), a.k.nu_code);
  }
  return (a.s1 * pe_min * mat / sqrt(rQ * T.rmin[ct]) + wt) * (1.0 + 1e-11);
}


// Exact d_r top-m over predecessors on spatial tiles.  CTA = one query tile (<= 64 rows of one time
// bucket, Morton order).  Candidate tiles are visited bucket by bucket backwards in time, each
// bucket outward from the tile nearest to the query tile; warp 0 tests 32 candidates at a time
// against the current thresholds (a bound that cannot beat the worst current list entry prunes the
// tile exactly), and the whole scan stops at the first bucket whose time lag alone prunes it.
// Survivors get the Gram W_Q^T W_C on the FP64 tensor pipe: mma.m8n8k4.f64 evaluates each element
// as the sequential fma chain over k (verified bit-identical on sm_100a, scripts/exp/dmma_order.cu),
// so G equals the oracle's chain exactly.  W chunks of kKC rows are staged by cp.async in a
// kStages ring; warp w owns the 16 x 32 sub-tile (rows 16 (w/2), cols 32 (w%2)).
constexpr size_t kDrStageDoubles = 2 * kQT * kKS;
// per-query lists of 32 LR slots (m_v <= 32 LR) follow the ring
constexpr size_t dr_smem(int LR) {
  return sizeof(double) * (kStages * kDrStageDoubles + kQT * 32 * LR) + sizeof(int) * kQT * 32 * LR;
}
static_assert(kStages * kDrStageDoubles >= kQT * (kCT + 1), "distance tile aliases the stages");

// Certified half-precision filter for one (query tile, candidate tile) pair.  G~ = W16_Q^T W16_C on
// the FP16 tensor pipe (mma.m16n8k16, f32 accumulate) bounds the exact chain G within
//   |G~ - G| <= 3e-3 |w_i||w_j| + 1e-5 (|w_i| + |w_j|)
// (inputs rounded to fp16: 2 * 2^-11 relative; f32 accumulation of <= 1024 products: 1024 * 2^-24 with
// a 16x margin for the tensor core's summation; the 2^8 prescale keeps values >= 2^-22 normal, and
// flushed ones contribute < 2^-22 each).  A pair can enter i's list only if the resulting lower bound
// of d_r does not exceed i's current worst entry; the tile is skipped when no pair can.  Block-wide
// (all threads), returns the same value in every thread.
constexpr int kHK = 64;        // halves per staged chunk
constexpr int kHS = kHK + 8;   // smem row stride (halves): conflict-free 32-bit fragment loads
static_assert(2 * kQT * kHS * 2 <= static_cast<int>(sizeof(double) * 2 * kQT * kKS), "half stage fits a ring slot");

__device__ __forceinline__ void ldsm_x4(const __half* p, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(a));
}

__device__ __forceinline__ void hmma_16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// diagnostics (STGP_DR_STATS): SM cycles per search phase, measured by thread 0 between the phase
// barriers, summed over CTAs into stats[50 + phase]
__device__ __forceinline__ void phase_clock(const DrArgs& a, long long& t, int slot) {
  if (!a.stats || threadIdx.x != 0) return;
  const long long now = clock64();
  atomicAdd(&a.stats[50 + slot], static_cast<unsigned long long>(now - t));
  t = now;
}

// Per-point data of a 64-row tile staged in shared memory (query tile once per CTA, candidate tile
// per tested pair): the pair tests and the d_r epilogue read these instead of scattered global loads.
struct TilePts {
  double x[kQT], y[kQT], r[kQT], rs[kQT], w[kQT];  // coordinates, residual r, 1 / sqrt(r), |w|
  int t[kQT], deg[kQT];                            // time id, degenerate flag
};
__device__ __forceinline__ void load_tile_pts(const DrArgs& a, int slot, int i, TilePts& P) {
  if (i < 0) {
    P.x[slot] = P.y[slot] = P.r[slot] = P.rs[slot] = P.w[slot] = 0.0;
    P.t[slot] = 0;
    P.deg[slot] = 1;
    return;
  }
  P.x[slot] = a.x[i];
  P.y[slot] = a.y[i];
  const double r = a.resid[i];
  P.r[slot] = r;
  P.rs[slot] = r > 0.0 ? 1.0 / sqrt(r) : 0.0;
  P.w[slot] = a.wnorm ? a.wnorm[i] : 0.0;  // set only with the fp16 filter (M > 0)
  P.t[slot] = a.tid[i];
  P.deg[slot] = a.degen[i];
}

// one_time: every query and candidate of the tile pair share one time each, so the temporal
// factors (pe1, pb1) are the pair's for every (i, j) -- no per-pair lag-table lookups.
template <int kL>
__device__ bool half_filter_survives(const DrArgs& a, double* ring, const int* qidx, const int* cidx, const int* qm,
                                     const double (*topd)[kL], const int (*topj)[kL], bool one_time, double pe1,
                                     double pb1, const TilePts& QP, const TilePts& CP, const int* qlive) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3, wr = wid >> 1, wc = wid & 1;
  float hc[4][4];
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int e = 0; e < 4; ++e) hc[v][e] = 0.f;
  long long tclk_f = a.stats ? clock64() : 0;
  const int nhc = a.ld16 / kHK;
  constexpr int kHPieces = 2 * kQT * (kHK / 8);  // 16-byte pieces per stage
  static_assert(kHPieces % kDrThreads == 0, "half staging split");
  auto stage = [&](int ch) {
    __half* hQ = reinterpret_cast<__half*>(ring + static_cast<size_t>(ch % kStages) * kDrStageDoubles);
    __half* hC = hQ + kQT * kHS;
#pragma unroll
    for (int it = 0; it < kHPieces / kDrThreads; ++it) {
      const int pc = tid + it * kDrThreads;
      const int which = pc / (kQT * (kHK / 8));
      const int rem = pc % (kQT * (kHK / 8));
      const int col = rem / (kHK / 8), piece = rem % (kHK / 8);
      const int g0 = which ? cidx[col] : qidx[col];
      const int g = g0 >= 0 ? g0 : 0;
      cp_async16((which ? hC : hQ) + col * kHS + 8 * piece,
                 a.W16 + static_cast<size_t>(g) * a.ld16 + static_cast<size_t>(ch) * kHK + 8 * piece);
    }
  };
#pragma unroll
  for (int ch = 0; ch < kStages - 1; ++ch) {
    if (ch < nhc) stage(ch);
    cp_async_commit();
  }
  for (int ch = 0; ch < nhc; ++ch) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (ch + kStages - 1 < nhc) stage(ch + kStages - 1);
    cp_async_commit();
    const __half* hQ = reinterpret_cast<const __half*>(ring + static_cast<size_t>(ch % kStages) * kDrStageDoubles);
    const __half* hC = hQ + kQT * kHS;
    // fragments by ldmatrix: one x4 for the 16 x 16 A block, two x4 for the four 8-candidate B blocks
    // (rows of 144 bytes: the eight row addresses of each 8 x 8 matrix fall in distinct bank groups)
    const __half* pa = hQ + (16 * wr + (lane & 15)) * kHS + (lane >> 4) * 8;
    const __half* pb = hC + (32 * wc + (lane >> 4) * 8 + (lane & 7)) * kHS + ((lane >> 3) & 1) * 8;
#pragma unroll
    for (int ks = 0; ks < kHK; ks += 16) {
      uint32_t a0, a1, a2, a3, b[8];
      ldsm_x4(pa + ks, a0, a1, a2, a3);
      ldsm_x4(pb + ks, b[0], b[1], b[2], b[3]);
      ldsm_x4(pb + 16 * kHS + ks, b[4], b[5], b[6], b[7]);
#pragma unroll
      for (int v = 0; v < 4; ++v) hmma_16816(hc[v], a0, a1, a2, a3, b[2 * v], b[2 * v + 1]);
    }
  }
  cp_async_wait<0>();
  if (a.stats) {  // diagnostics: the fp16 Gram part of the filter (slot 6); the pair test follows
    __syncthreads();
    phase_clock(a, tclk_f, 6);
  }
  // pair test: can (i, j) still enter i's list?  k(i, j) in single precision with the fast exp:
  // |k_f - k| <= 1e-5 |k_f| + 1e-30 covers its ~10 roundings and the 2-ulp __expf (rel. ~1.3e-6).
  int surv = a.k.nu_code == kNuGeneral ? 1 : 0;  // no single-precision general Matern: all go exact
  constexpr double kUnscale = 1.0 / (kW16Scale * kW16Scale);
  const float cf = static_cast<float>(a.k.c), s1f = static_cast<float>(a.k.s1);
  int iq[2];
  float xq[2], yq[2], rsq[2], wq[2], dwq2[2];  // rsq: 1 / sqrt(r_i); dwq2: current worst d^2
  double dwq[2];
  int tq[2], mq[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int qq = 16 * wr + grp + 8 * h;
    const int i = qidx[qq];
    const int m = qlive[qq] ? qm[qq] : 0;  // a query the live test excluded takes none of the tile
    iq[h] = i;
    mq[h] = m;
    if (i >= 0) {
      xq[h] = static_cast<float>(QP.x[qq]);
      yq[h] = static_cast<float>(QP.y[qq]);
      tq[h] = QP.t[qq];
      rsq[h] = static_cast<float>(QP.rs[qq]);
      wq[h] = static_cast<float>(QP.w[qq]);
      dwq[h] = m > 0 ? topd[qq][m - 1] : 0.0;
      dwq2[h] = static_cast<float>(fmin(dwq[h], 1.0) * fmin(dwq[h], 1.0));
    }
  }
#pragma unroll
  for (int v = 0; v < 4; ++v)
#pragma unroll
    for (int e2 = 0; e2 < 2; ++e2) {
      const int cc = 32 * wc + 8 * v + 2 * tig + e2;
      const int j = cidx[cc];
      if (j < 0 || surv) continue;
      const bool dj = CP.deg[cc] != 0;
      const float xj = static_cast<float>(CP.x[cc]), yj = static_cast<float>(CP.y[cc]);
      const int tj = CP.t[cc];
      // 1 / sqrt(r_i r_j) as a product of rounded reciprocal roots: a few ulp below the exact value at
      // most, far inside the bound's (1 + 1e-12) margin
      const float rsj = static_cast<float>(CP.rs[cc]), wj = static_cast<float>(CP.w[cc]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = iq[h], m = mq[h];
        if (i < 0 || j >= i || m <= 0) continue;
        const double dw = dwq[h];
        if (dj) {  // d = 1 exactly
          if (lex_less(1.0, j, dw, topj[16 * wr + grp + 8 * h][m - 1])) surv = 1;
          continue;
        }
        double pe = pe1, pb = pb1;
        if (!one_time) a.lt.get2(tq[h], tj, pe, pb);
        const float dx = xq[h] - xj, dy = yq[h] - yj;
        const float xm = cf * sqrtf(dx * dx + dy * dy) * static_cast<float>(pb);
        const float ex = __expf(-xm);
        const float mat = a.k.nu_code == 0 ? ex : (a.k.nu_code == 1 ? (1.f + xm) * ex : (1.f + xm + xm * xm * (1.f / 3.f)) * ex);
        // the bound in single precision: the difference kf - g loses at most ~2^-23 (|kf| + |g|)
        // (covered by the 1e-6 (|kf| + |g|) term), the products and sums ~10 roundings of 2^-24
        // (the 4e-6 relative margin), the final comparison the 1e-6 absolute one (d^2 <= 1)
        const float kf = s1f * static_cast<float>(pe) * mat;
        const float g = hc[v][2 * h + e2] * static_cast<float>(kUnscale);
        const float err = 3e-3f * wq[h] * wj + 1e-5f * (wq[h] + wj) + 1e-5f * fabsf(kf) +
                          1e-6f * (fabsf(kf) + fabsf(g)) + 1e-30f;
        const float ub = ((fabsf(kf - g) + err) * rsq[h] * rsj) * (1.0f + 4e-6f);
        if (!((1.0f - ub) - 1e-6f > dwq2[h])) surv = 1;
      }
    }
  return __syncthreads_or(surv) != 0;
}

template <bool GEN, int LR>  // GEN: general nu; LR: list slots per lane (m_v <= 32 LR)
__global__ void __launch_bounds__(kDrThreads, 2) knn_dr_kernel(DrArgs a) {  // 2 CTAs per SM (128 registers)
  constexpr int kL = 32 * LR;
  extern __shared__ double sm[];
  // the staging ring and the distance tile are never live together
  double* ring = sm;
  double (*sd)[kCT + 1] = reinterpret_cast<double (*)[kCT + 1]>(sm);
  double (*topd)[kL] = reinterpret_cast<double (*)[kL]>(sm + kStages * kDrStageDoubles);
  int (*topj)[kL] = reinterpret_cast<int (*)[kL]>(sm + kStages * kDrStageDoubles + kQT * kL);
  __shared__ int qidx[kQT], cidx[kCT], qm[kQT], qemit[kQT];
  __shared__ TilePts sQP, sCP;
  __shared__ double s_dmax[kDrThreads / 32];
  __shared__ int s_surv[32], s_nsurv;
  __shared__ double s_wt[32], s_pemin[32], s_pbmax[32];  // tile_pair_terms of each surviving tile
  __shared__ int s_qlive[kQT];  // per-query live test of the current candidate tile (1: may take one)
  __shared__ double s_d;
  __shared__ double sAQ[kMaxGroups];
  const DrTiles& T = a.T;
  const int qt = a.tile0 + blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  const int wr = wid >> 1, wc = wid & 1;  // warp sub-tile: rows 16 wr.., cols 32 wc..
  for (int e = tid; e < kQT * kL; e += kDrThreads) {
    topd[e / kL][e % kL] = __longlong_as_double(0x7ff0000000000000LL);
    topj[e / kL][e % kL] = INT_MAX;
  }
  const int qp0 = T.off[qt], qn = T.off[qt + 1] - qp0;
  if (tid < kQT) {
    const int i = tid < qn ? T.sp[qp0 + tid] : -1;
    qidx[tid] = i;
    qemit[tid] = i >= 0 ? min(a.m_v, i) : 0;
    // a degenerate query has d = 1 to every predecessor: its list is the m smallest indices
    qm[tid] = (i >= 0 && !a.degen[i]) ? min(a.m_v, i) : 0;
    STGP_DCHECK(qemit[tid] <= kL);
    load_tile_pts(a, tid, i, sQP);
  }
  for (int g = tid; g < T.G; g += kDrThreads) sAQ[g] = T.A[static_cast<size_t>(qt) * T.G + g];
  __syncthreads();
  for (int e = tid; e < kQT * kL; e += kDrThreads) {
    const int qq = e / kL, l = e % kL, i = qidx[qq];
    if (i >= 0 && a.degen[i] && l < qemit[qq]) {
      topd[qq][l] = 1.0;
      topj[qq][l] = l;
    }
  }
  const int qb = T.bucket[qt];
  const int tminQ = T.tmin[qt], tmaxQ = T.tmax[qt], imaxQ = T.imax[qt];
  const double qx0 = T.bx0[qt], qx1 = T.bx1[qt], qy0 = T.by0[qt], qy1 = T.by1[qt];
  const double rQ = T.rmin[qt];
  const bool can_prune = a.prune != 0;
  const uint32_t qkey = T.key[qt];
  const int nch = a.ldm / kKC;
  constexpr int kPieces = 2 * kQT * (kKC / 2);  // Q and C, 16 B each
  static_assert(kPieces % kDrThreads == 0, "staging split");
  __syncthreads();

  // phase 0 seeds the lists with the 2 kSeed + 1 nearest tiles of this and the previous bucket
  // (queries early in their bucket have few same-bucket predecessors, so thresholds would stay
  // infinite through the whole same-bucket scan); phase 1 is the pruned traversal, skipping seeds.
  constexpr int kSeed = 1;
  for (int phase = 0; phase < 2; ++phase)
  for (int b = qb; b >= 0; --b) {
    if (phase == 0 && b < qb - 1) break;
    const int t0 = T.b_tile0[b], t1 = T.b_tile0[b + 1];
    int p = qt;
    if (b != qb) {  // nearest tile by Morton key
      int lo = t0, hi = t1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (T.key[mid] < qkey) lo = mid + 1; else hi = mid;
      }
      p = min(lo, t1 - 1);
    }
    const int R = max(p - t0, t1 - 1 - p);
    const bool seeded = b >= qb - 1;
    const int s_first = (phase == 1 && seeded) ? 2 * kSeed + 1 : 0;
    const int s_last = phase == 0 ? min(2 * kSeed, 2 * R) : 2 * R;
    bool stop = false;
    for (int s0 = s_first; s0 <= s_last && !stop; s0 += 32) {
      long long tclk = a.stats ? clock64() : 0;
      // current worst threshold over the tile's queries (inf while any list is short)
      {
        double dm = 0.0;
        for (int qq = tid; qq < kQT; qq += kDrThreads)
          if (qm[qq] > 0) dm = fmax(dm, topd[qq][qm[qq] - 1]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(kFull, dm, o));
        if (lane == 0) s_dmax[wid] = dm;
        __syncthreads();
        if (tid == 0) {
          double d = 0.0;
          for (int w2 = 0; w2 < kDrThreads / 32; ++w2) d = fmax(d, s_dmax[w2]);
          s_d = d;
        }
        __syncthreads();
      }
      const double d = s_d;
      if (wid == 0) {
        // bucket-level stop: the time lag alone prunes this and every earlier bucket
        bool stop_b = false;
        if (phase == 1 && can_prune && b != qb && s0 == s_first && d < 1.0) {
          double pe, pb;
          a.lt.get2(tminQ, T.b_tmax[b], pe, pb);
          double wt = 0.0;
          const double* Ab = T.Apre + static_cast<size_t>(b) * T.G;
          for (int g = 0; g < T.G; ++g) wt += sAQ[g] * Ab[g];
          const double cb = (a.s1 * pe / sqrt(rQ * T.rpre[b]) + wt) * (1.0 + 1e-11);
          stop_b = cb < 1.0 && (1.0 - cb) - 1e-12 > d * d;
        }
        const int s = s0 + lane;
        const int off = (s & 1) ? -((s + 1) >> 1) : (s >> 1);
        const int ct = p + off;
        bool take = !stop_b && s <= s_last && ct >= t0 && ct < t1 && T.imin[ct] < imaxQ;
        int pruned = 0;
        double pe_min = 1.0, pb_max = 1.0, wt = 0.0;
        if (take && phase == 1 && can_prune) tile_pair_terms(a, tminQ, tmaxQ, sAQ, ct, pe_min, pb_max, wt);
        if (take && phase == 1 && can_prune && d < 1.0) {
          const double cmax = tile_cmax(a, qx0, qx1, qy0, qy1, rQ, ct, pe_min, pb_max, wt);
          if (cmax < 1.0 && (1.0 - cmax) - 1e-12 > d * d) {
            take = false;
            pruned = 1;
          }
        }
        const unsigned mk = __ballot_sync(kFull, take);
        if (take) {
          const int pos = __popc(mk & ((1u << lane) - 1));
          s_surv[pos] = ct;
          s_wt[pos] = wt;
          s_pemin[pos] = pe_min;
          s_pbmax[pos] = pb_max;
        }
        if (lane == 0) {
          s_nsurv = stop_b ? -1 : __popc(mk);
          if (a.stats) {
            atomicAdd(&a.stats[0], static_cast<unsigned long long>(__popc(mk)));
            const int lg = min(qb - b, 15);
            atomicAdd(&a.stats[2 + lg], static_cast<unsigned long long>(__popc(mk)));
            if (stop_b) atomicAdd(&a.stats[34 + lg], 1ull);
          }
        }
        if (a.stats) {
          const unsigned pk = __ballot_sync(kFull, pruned);
          if (lane == 0 && pk) {
            atomicAdd(&a.stats[1], static_cast<unsigned long long>(__popc(pk)));
            atomicAdd(&a.stats[18 + min(qb - b, 15)], static_cast<unsigned long long>(__popc(pk)));
          }
        }
      }
      __syncthreads();
      phase_clock(a, tclk, 0);  // tile selection
      const int nsurv = s_nsurv;
      if (nsurv < 0) {
        stop = true;
        break;
      }
      for (int sv = 0; sv < nsurv; ++sv) {
        const int ct = s_surv[sv];
        if (tid < kQT) s_qlive[tid] = 1;  // (the live test below narrows it; visible after the next barrier)
        if (phase == 1 && can_prune) {
          // per-query re-test with each row's own threshold, time, point-to-box distance and r
          // (the tile-level test above used the worst of 64 of each): a valid bound per pair, the
          // tile is skipped when no query row can take any of its candidates
          int live = 0;
          if (tid < kQT) {
            const int qq = tid, m = qm[qq];
            if (m > 0) {
              const double dq = topd[qq][m - 1];
              if (!(dq < 1.0)) {
                live = 1;
              } else {
                double pe_min = s_pemin[sv], pb_max = s_pbmax[sv];  // the query tile's, exact when it has
                if (tminQ != tmaxQ) {                               // one time; else each row's own
                  const int ti = sQP.t[qq], tc0 = T.tmin[ct], tc1 = T.tmax[ct];
                  double pb0, pe0;
                  if (tc1 >= ti) pe_min = 1.0; else a.lt.get2(ti, tc1, pe_min, pb0);
                  a.lt.get2(ti, tc0, pe0, pb_max);
                }
                double mat = 1.0;
                if (a.k.nu_code != kNuGeneral) {
                  const double xi = sQP.x[qq], yi = sQP.y[qq];
                  const double dx = fmax(0.0, fmax(T.bx0[ct] - xi, xi - T.bx1[ct]));
                  const double dy = fmax(0.0, fmax(T.by0[ct] - yi, yi - T.by1[ct]));
                  const double xm = a.k.c * sqrt(dx * dx + dy * dy) * (1.0 - 1e-12) * pb_max * (1.0 - 1e-12);
                  mat = matern_from_exp(xm, exp(-xm), a.k.nu_code);
                }
                const double ci = (a.s1 * pe_min * mat / sqrt(sQP.r[qq] * T.rmin[ct]) + s_wt[sv]) * (1.0 + 1e-11);
                live = !(ci < 1.0 && (1.0 - ci) - 1e-12 > dq * dq);
              }
            }
          }
          if (tid < kQT) s_qlive[tid] = live;
          const int any = __syncthreads_or(live);
          phase_clock(a, tclk, 1);  // per-query live test
          if (!any) {
            if (a.stats && tid == 0) {
              atomicAdd(&a.stats[0], ~0ull);  // -1: moved from evaluated to pruned
              atomicAdd(&a.stats[1], 1ull);
              atomicAdd(&a.stats[2 + min(qb - b, 15)], ~0ull);
              atomicAdd(&a.stats[18 + min(qb - b, 15)], 1ull);
            }
            continue;
          }
        }
        const int cp0 = T.off[ct], cn = T.off[ct + 1] - cp0;
        // single-time query and candidate tiles (the common case: buckets are days): one lag-table
        // entry serves every pair of the tile pair
        const bool one_time = tminQ == tmaxQ && T.tmin[ct] == T.tmax[ct];
        double pe1 = 1.0, pb1 = 1.0;
        if (one_time) a.lt.get2(tminQ, T.tmin[ct], pe1, pb1);
        if (tid < kCT) {
          const int j = tid < cn ? T.sp[cp0 + tid] : -1;
          cidx[tid] = j;
          load_tile_pts(a, tid, j, sCP);
        }
        __syncthreads();
        if (a.W16 && phase == 1 && a.M > 0) {  // certified half-precision filter (seeds run exactly)
          const bool fs = half_filter_survives(a, ring, qidx, cidx, qm, topd, topj, one_time, pe1, pb1, sQP, sCP, s_qlive);
          phase_clock(a, tclk, 2);  // half-precision filter
          if (!fs) {
            if (a.stats && tid == 0) atomicAdd(&a.stats[47], 1ull);
            continue;
          }
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
              const int g0 = which ? cidx[col] : qidx[col];
              const int g = g0 >= 0 ? g0 : 0;  // padding columns: any row, never read back
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
        phase_clock(a, tclk, 3);  // exact Gram (staging + DMMA)
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int qq = 16 * wr + 8 * u + grp, cc = 32 * wc + 8 * v + 2 * tig + h;
              const int i = qidx[qq], j = cidx[cc];
              double dd = __longlong_as_double(0x7ff0000000000000LL);
              if (i >= 0 && j >= 0 && j < i) {
                if (sQP.deg[qq] || sCP.deg[cc]) {
                  dd = 1.0;
                } else {
                  double pe = pe1, pb = pb1;  // the same table entry as a per-pair lookup
                  if (!one_time) a.lt.get2(sQP.t[qq], sCP.t[cc], pe, pb);
                  TF f;
                  f.pow_mE = pe;
                  f.pow_mbh = pb;
                  double rho = gneiting_eval<GEN>(a.k, spatial_dist(sQP.x[qq], sQP.y[qq], sCP.x[cc], sCP.y[cc]), f);
                  if (a.M > 0) rho = __dsub_rn(rho, acc[u][v][h]);
                  const double rad =
                      __dsub_rn(1.0, __ddiv_rn(fabs(rho), __dsqrt_rn(__dmul_rn(sQP.r[qq], sCP.r[cc]))));
                  dd = __dsqrt_rn(rad < 0.0 ? 0.0 : rad);
                }
              }
              sd[qq][cc] = dd;
            }
        __syncthreads();
        phase_clock(a, tclk, 4);  // d_r epilogue
        // merge: warp wid handles queries wid, wid + 8, ...
        bool inserted = false;
        for (int qq = wid; qq < kQT; qq += kDrThreads / 32) {
          const int i = qidx[qq];
          const int m = qm[qq];
          if (m <= 0) continue;
          TopM e[LR];
#pragma unroll
          for (int r = 0; r < LR; ++r) e[r] = TopM{topd[qq][32 * r + lane], topj[qq][32 * r + lane]};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = lane + 32 * h;
            const int j = cidx[cc];
            const double dd = sd[qq][cc];
            double wd;
            int wj;
            topl_worst(e, m, wd, wj);
            const unsigned acc2 = __ballot_sync(kFull, j >= 0 && j < i && lex_less(dd, j, wd, wj));
            if (acc2) {
              topl_insert(e, m, acc2, dd, j, lane);
              inserted = true;
            }
          }
#pragma unroll
          for (int r = 0; r < LR; ++r) {
            topd[qq][32 * r + lane] = e[r].d;
            topj[qq][32 * r + lane] = e[r].j;
          }
        }
        if (a.stats) {  // diagnostics: evaluated tiles that changed some list
          const int any = __syncthreads_or(inserted ? 1 : 0);
          if (tid == 0 && any) atomicAdd(&a.stats[48 + phase], 1ull);
        }
        __syncthreads();
        phase_clock(a, tclk, 5);  // list merge
      }
    }
    if (stop) break;
  }
  __syncthreads();
  for (int qq = wid; qq < kQT; qq += kDrThreads / 32) {
    const int i = qidx[qq];
    if (i < 0) continue;
    const int m = qemit[qq];
    TopM e[LR];
#pragma unroll
    for (int r = 0; r < LR; ++r) e[r] = TopM{topd[qq][32 * r + lane], topj[qq][32 * r + lane]};
    topl_emit(e, a.m_v, m, lane, a.out + static_cast<size_t>(i) * a.m_v,
              a.dist ? a.dist + static_cast<size_t>(i) * a.m_v : nullptr);
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

}  // extern "C"

namespace stgp {

// The exact spatial-tile search over predecessors (header comments of knn_dr_kernel).  With
// inducing points it is the d_r search (neighbors.cpp:51-83, 324-329); with none, r_i = s1 and
// w = 0, so d = sqrt(1 - |k| / sqrt(s1 s1)) = sqrt(1 - |k / s1|) (sqrt(fl(s1 s1)) = s1 in round to
// nearest): the d_c search (neighbors.cpp:37-43, 318-322), pruned spatially instead of by time only.
stgp_neighbors* spatial_search(stgp_dataset* ds, const Params& p, const std::vector<double>& zxyt, int m_v,
                               int kind) {
  stgp_neighbors* result = nullptr;
  auto frees_clk = std::chrono::steady_clock::now();
  {
    if (m_v < 0) config_error("m_v must be >= 0");
    if (m_v > kMaxSearchM) config_error("neighbour search supports m_v <= 128 on the device");
    stgp_ctx* ctx = ds->ctx;
    cudaStream_t st = ctx->stream;
    const int n = ds->n, M = static_cast<int>(zxyt.size() / 3);
    const DevKernel k = dev_kernel(p);
    // diagnostics (STGP_DR_STATS): host-side phase times
    const bool dbg = std::getenv("STGP_DR_STATS") != nullptr;
    const bool host_laps = std::getenv("STGP_DR_HOSTLAPS") != nullptr;  // host-side time per phase, no sync
    auto clk0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!dbg && !host_laps) return;
      if (dbg) STGP_CUDA(cudaStreamSynchronize(st));
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[stgp] d_r phase %-12s %8.2f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - clk0).count());
      clk0 = now;
    };
    // time index over data + inducing times, live factors (no lag table in the selection kernel)
    std::vector<double> zx(M), zy(M), zt(M);
    for (int j = 0; j < M; ++j) {
      zx[j] = zxyt[3 * j];
      zy[j] = zxyt[3 * j + 1];
      zt[j] = zxyt[3 * j + 2];
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
    lap("setup");
    // W lives in the context between searches: an 8 GB cudaMalloc / cudaFree per call costs 0.1-1 s
    DevBuf<double>& W = ctx->sel_W;
    // column slab of each rank's whitening (a multiple of the 64-column block; world slabs cover n)
    const int wcols = ctx->world > 1 ? ceil_div(ceil_div(n, ctx->world), kWB) * kWB : n;
    W.ensure(static_cast<size_t>(ldm) * std::max<long long>(n, static_cast<long long>(wcols) * ctx->world));
    DevBuf<double> resid(n), wnorm(n);
    lap("alloc W");
    STGP_CUDA(cudaMemsetAsync(W.get(), 0, sizeof(double) * ldm * n, st));
    DevBuf<int32_t> degen(n);
    // basis buffers live to the end of the search: freeing them here (cudaFree synchronizes the device)
    // would hold the host until the whitening finishes instead of overlapping the tile set-up with it
    DevBuf<double> A, L, Lp;
    DevBuf<int> fail;
    {
      lap("setup+alloc");
      ProfRegion pr(ctx, "dr_whiten");
      if (M > 0) {
        // InducingBasis(set, selection kernel): jittered Sigma_m, one retry at 10x (inducing.cpp:250-261)
        A.alloc(static_cast<size_t>(M) * M);
        L.alloc(static_cast<size_t>(M) * M);
        fail.alloc(1);
        const double jitter = 1e-8 * p.sigma1_2;
        bool ok = false;

        for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
          std::unique_ptr<ProfRegion> prc(new ProfRegion(ctx, "dr_sigma_chol"));
          sel_sigma_kernel<<<grid_for(static_cast<long long>(M) * M), 256, 0, st>>>(
              dzx.get(), dzy.get(), dzt.get(), M, k, lt, jitter, attempt == 0 ? 0.0 : 9.0 * jitter, A.get());
          launched(ctx);
          fail.zero(st);
          for (int j0 = 0; j0 < M; j0 += kCP) {
            const int pw = std::min(kCP, M - j0);
            chol_panel_update_kernel<<<ceil_div(M - j0, 64), 128, 0, st>>>(A.get(), M, j0, pw, L.get());
            chol_panel_factor_kernel<<<1, 1024, 0, st>>>(M, j0, pw, L.get(), fail.get());
            ctx->launches += 1;
          }
          launched(ctx);
          prc.reset();
          int f = 0;
          fail.download(&f, 1, st);
          STGP_CUDA(cudaStreamSynchronize(st));
          ok = f == 0;
        }
        if (!ok) numeric_error("InducingBasis: inducing covariance is not positive definite");
        lap("w:sigma+chol");
        auto wkern = k.nu_code == kNuGeneral ? whiten_seq_kernel<true> : whiten_seq_kernel<false>;
        STGP_CUDA(cudaFuncSetAttribute(wkern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kWsmem)));
        const int ldL = (M + kWKC - 1) / kWKC * kWKC;
        Lp.alloc(static_cast<size_t>(M) * ldL);
        ProfRegion prw(ctx, "dr_whiten_seq");
        pad_rows_kernel<<<grid_for(static_cast<long long>(M) * ldL), 256, 0, st>>>(L.get(), M, ldL, Lp.get());
        launched(ctx);
        // sharded: each rank whitens its slab of wcols columns, then the slabs are all-gathered
        // (columns are independent, so the gathered W equals one rank's full whitening bit for bit)
        const int w0 = std::min(n, ctx->rank * wcols), w1 = std::min(n, w0 + wcols);
        if (w1 > w0)
          wkern<<<ceil_div(w1 - w0, kWB), kWthreads, kWsmem, st>>>(dzx.get(), dzy.get(), dzt.get(), M, ldm,
                                                                    ds->x.get(), ds->y.get(), ds->tid.get(), w0, w1, k,
                                                                    lt, Lp.get(), ldL, W.get());
        launched(ctx);
        if (ctx->world > 1) allgather_cols(ctx, W.get(), static_cast<size_t>(ldm) * wcols, n, ldm);
        lap("w:whiten_seq");
      }
      ProfRegion prr(ctx, "dr_resid");
      resid_kernel<<<std::max(1, std::min(ceil_div(n, kResRows), ctx->num_sms * 16)), kResRows, 0, st>>>(
          W.get(), M, ldm, n, p.sigma1_2, resid.get(), degen.get(), wnorm.get());
      launched(ctx);
    }
    lap("whiten");
    auto nb = std::make_unique<stgp_neighbors>();
    nb->ctx = ctx;
    nb->n = n;
    nb->m_v = std::max(m_v, 1);
    nb->kind = kind;
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
      // certified half-precision filter (STGP_DR_FILTER=0 disables): fp16 copy of W, |w| bounds
      if (M > 0 && !(std::getenv("STGP_DR_FILTER") && std::getenv("STGP_DR_FILTER")[0] == '0')) {
        const int ld16 = (M + kHK - 1) / kHK * kHK;
        ctx->sel_W16.ensure(static_cast<size_t>(ld16) * n);
        __half* w16 = reinterpret_cast<__half*>(ctx->sel_W16.get());
        w16_kernel<<<grid_for(static_cast<long long>(ld16) * n, 256, ctx->num_sms * 32), 256, 0, st>>>(W.get(), M, ldm, n,
                                                                                                      ld16, w16);
        launched(ctx);
        a.W16 = w16;
        a.ld16 = ld16;
        a.wnorm = wnorm.get();
      }
      a.tid = ds->tid.get();
      a.degen = degen.get();
      a.k = k;
      a.lt = lt;
      a.out = nb->idx.get();
      a.dist = nb->dist.get();
      // spatial tiles: time buckets (consecutive equal-time blocks merged to >= 64 rows) sorted by
      // the Morton code of (x, y), cut into tiles of <= 64 rows; one index-order bucket when the rows
      // are not time sorted (no pruning: plain exact brute force over predecessors).
      const bool ts = ds->time_sorted;
      std::unique_lock<std::mutex> meta_lock(ds->tile_mu);
      if (!ds->tile_meta) {  // per dataset (immutable): bucket starts and bounding box
        std::vector<int>& bs = ds->tile_bstart;
        bs.assign(1, 0);
        if (ts) {
          int cnt = 0;
          for (int i = 0; i < n; ++i) {
            if (i > 0 && ds->htid[static_cast<size_t>(i)] != ds->htid[static_cast<size_t>(i - 1)] && cnt >= kQT) {
              bs.push_back(i);
              cnt = 0;
            }
            ++cnt;
          }
        }
        bs.push_back(n);
        double bx0 = INFINITY, bx1 = -INFINITY, by0 = INFINITY, by1 = -INFINITY;
        for (int i = 0; i < n; ++i) {
          bx0 = std::min(bx0, ds->hx[i]);
          bx1 = std::max(bx1, ds->hx[i]);
          by0 = std::min(by0, ds->hy[i]);
          by1 = std::max(by1, ds->hy[i]);
        }
        ds->tile_x0 = bx0;
        ds->tile_x1 = bx1;
        ds->tile_y0 = by0;
        ds->tile_y1 = by1;
        ds->tile_meta = true;
      }
      meta_lock.unlock();  // written once, read-only from here on
      const std::vector<int>& bstart = ds->tile_bstart;
      const int nbucket = static_cast<int>(bstart.size()) - 1;
      const double x0 = ds->tile_x0, x1 = ds->tile_x1, y0 = ds->tile_y0, y1 = ds->tile_y1;
      const double sx = x1 > x0 ? 65535.0 / (x1 - x0) : 0.0, sy = y1 > y0 ? 65535.0 / (y1 - y0) : 0.0;
      // rows sorted by (bucket, Morton key) on the device: a stable radix sort keeps index order
      // within equal keys; the keys are formed on the device (the host loop cost ~7 ms at cfg4)
      std::unique_ptr<uint64_t[]> key64(new uint64_t[static_cast<size_t>(n)]);  // filled by the download below
      lap("tiles:keys");
      DevBuf<int32_t> d_sp;
      DevBuf<uint64_t> d_keys_sorted;
      {
        DevBuf<uint64_t> d_keys(static_cast<size_t>(n));
        DevBuf<int32_t> d_iota(static_cast<size_t>(n)), d_bstart;
        d_bstart.upload(bstart.data(), bstart.size(), st);
        tile_keys_kernel<<<grid_for(n, 256, ctx->num_sms * 8), 256, 0, st>>>(n, ds->x.get(), ds->y.get(), d_bstart.get(),
                                                                           nbucket, ts, x0, y0, sx, sy, d_keys.get(),
                                                                           d_iota.get());
        launched(ctx);
        lap("tiles:upload");
        d_sp.alloc(static_cast<size_t>(n));
        d_keys_sorted.alloc(static_cast<size_t>(n));
        const int endbit = 32 + std::max(1, static_cast<int>(std::ceil(std::log2(static_cast<double>(nbucket) + 1.0))));
        size_t tmpb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmpb, d_keys.get(), d_keys_sorted.get(), d_iota.get(), d_sp.get(), n,
                                        0, std::min(64, endbit), st);
        DevBuf<unsigned char> tmp(tmpb);
        lap("tiles:sortq");
        cub::DeviceRadixSort::SortPairs(tmp.get(), tmpb, d_keys.get(), d_keys_sorted.get(), d_iota.get(), d_sp.get(),
                                        n, 0, std::min(64, endbit), st);
        launched(ctx);
        lap("tiles:sort");
        d_keys_sorted.download(key64.get(), static_cast<size_t>(n), st);  // sorted keys: tile anchors
        STGP_CUDA(cudaStreamSynchronize(st));
      }
      std::vector<int32_t> toff, tbucket, btile0;
      std::vector<uint32_t> tkey;
      for (int bb = 0; bb < nbucket; ++bb) {
        const int b0 = bstart[static_cast<size_t>(bb)], b1 = bstart[static_cast<size_t>(bb) + 1];
        btile0.push_back(static_cast<int32_t>(toff.size()));
        for (int q = b0; q < b1; q += kQT) {
          toff.push_back(q);
          tbucket.push_back(bb);
          tkey.push_back(static_cast<uint32_t>(key64[static_cast<size_t>(q)] & 0xffffffffu));
        }
      }
      const int ntile = static_cast<int>(toff.size());
      toff.push_back(n);
      btile0.push_back(ntile);
      DevBuf<int32_t> d_off, d_bucket, d_bt0, d_btmax;
      DevBuf<uint32_t> d_key;
      d_off.upload(toff.data(), toff.size(), st);
      d_bucket.upload(tbucket.data(), tbucket.size(), st);
      d_bt0.upload(btile0.data(), btile0.size(), st);
      d_key.upload(tkey.data(), tkey.size(), st);
      DevBuf<int> tmn(ntile), tmx(ntile), hdg(ntile), imn(ntile), imx(ntile);
      DevBuf<double> wmx(ntile), rmn(ntile), bx0(ntile), bx1(ntile), by0(ntile), by1(ntile);
      DrTiles T{};
      T.sp = d_sp.get();
      T.off = d_off.get();
      T.bucket = d_bucket.get();
      T.b_tile0 = d_bt0.get();
      T.key = d_key.get();
      T.tmin = tmn.get();
      T.tmax = tmx.get();
      T.hasdeg = hdg.get();
      T.imin = imn.get();
      T.imax = imx.get();
      T.bx0 = bx0.get();
      T.bx1 = bx1.get();
      T.by0 = by0.get();
      T.by1 = by1.get();
      T.wmax = wmx.get();
      T.rmin = rmn.get();
      tile_stats_kernel<<<ntile, 64, 0, st>>>(T, ds->x.get(), ds->y.get(), resid.get(), degen.get(), ds->tid.get(),
                                              p.sigma1_2);
      launched(ctx);
      lap("tiles");
      // inducing-point groups for the block-norm bound: inducing time (<= 4 bins) x spatial cell
      // (<= 12 cells of the inducing bounding box)
      int G = 0;
      std::vector<int32_t> kgroup(static_cast<size_t>(std::max(M, 1)), 0);
      if (M > 0) {
        const int gt = std::min<int>(4, static_cast<int>(Ti.size()));
        double zx0 = INFINITY, zx1 = -INFINITY, zy0 = INFINITY, zy1 = -INFINITY;
        for (int j = 0; j < M; ++j) {
          zx0 = std::min(zx0, zx[j]);
          zx1 = std::max(zx1, zx[j]);
          zy0 = std::min(zy0, zy[j]);
          zy1 = std::max(zy1, zy[j]);
        }
        const double ex = std::max(zx1 - zx0, 1e-300), ey = std::max(zy1 - zy0, 1e-300);
        int gx = std::max(1, std::min(12, static_cast<int>(std::lround(std::sqrt(12.0 * ex / ey)))));
        int gy = std::max(1, 12 / gx);
        G = gt * gx * gy;
        for (int j = 0; j < M; ++j) {
          const int ti_ = static_cast<int>(std::lower_bound(Ti.begin(), Ti.end(), zt[j]) - Ti.begin());
          const int tg = static_cast<int>(static_cast<long long>(ti_) * gt / static_cast<long long>(Ti.size()));
          const int cx = std::min(gx - 1, static_cast<int>((zx[j] - zx0) / ex * gx));
          const int cy = std::min(gy - 1, static_cast<int>((zy[j] - zy0) / ey * gy));
          kgroup[static_cast<size_t>(j)] = (tg * gy + cy) * gx + cx;
        }
      }
      DevBuf<int32_t> d_kgroup;
      d_kgroup.upload(kgroup.data(), kgroup.size(), st);
      DevBuf<double> dA(static_cast<size_t>(std::max(1, ntile * G)));
      T.G = G;
      T.A = dA.get();
      if (G > 0) {
        tile_groups_kernel<<<ntile, 256, 0, st>>>(T, W.get(), ldm, M, d_kgroup.get(), resid.get(), degen.get());
        launched(ctx);
      }
      // per-bucket prefix bounds (buckets <= b) for the exact early stop (host, small)
      std::vector<double> hA(static_cast<size_t>(ntile) * G), hr(static_cast<size_t>(ntile));
      std::vector<int> htmax(static_cast<size_t>(ntile));
      if (G > 0) dA.download(hA.data(), hA.size(), st);
      rmn.download(hr.data(), hr.size(), st);
      tmx.download(htmax.data(), htmax.size(), st);
      STGP_CUDA(cudaStreamSynchronize(st));
      std::vector<double> Apre(std::max<size_t>(static_cast<size_t>(nbucket) * G, 1), 0.0), rpre(static_cast<size_t>(nbucket), INFINITY);
      std::vector<int32_t> btmax(static_cast<size_t>(nbucket), -1);
      for (int t2 = 0; t2 < ntile; ++t2) {
        const size_t bb = static_cast<size_t>(tbucket[static_cast<size_t>(t2)]);
        btmax[bb] = std::max(btmax[bb], htmax[static_cast<size_t>(t2)]);
        rpre[bb] = std::min(rpre[bb], hr[static_cast<size_t>(t2)]);
        for (int g = 0; g < G; ++g)
          Apre[bb * G + g] = std::max(Apre[bb * G + g], hA[static_cast<size_t>(t2) * G + g]);
      }
      for (int bb = 1; bb < nbucket; ++bb) {
        rpre[static_cast<size_t>(bb)] = std::min(rpre[static_cast<size_t>(bb)], rpre[static_cast<size_t>(bb) - 1]);
        for (int g = 0; g < G; ++g)
          Apre[static_cast<size_t>(bb) * G + g] =
              std::max(Apre[static_cast<size_t>(bb) * G + g], Apre[static_cast<size_t>(bb - 1) * G + g]);
      }
      DevBuf<double> dApre, drpre;
      dApre.upload(Apre.data(), Apre.size(), st);
      drpre.upload(rpre.data(), rpre.size(), st);
      d_btmax.upload(btmax.data(), btmax.size(), st);
      T.b_tmax = d_btmax.get();
      T.Apre = dApre.get();
      T.rpre = drpre.get();
      a.T = T;
      a.s1 = p.sigma1_2;
      // pruning needs time-sorted rows (tile time ranges); otherwise plain brute force
      a.prune = ts ? 1 : 0;
      lap("groups");
      DevBuf<unsigned long long> stats;
      if (std::getenv("STGP_DR_STATS")) {  // diagnostics: tile pairs evaluated / pruned
        stats.alloc(64);
        STGP_CUDA(cudaMemsetAsync(stats.get(), 0, 64 * 8, st));
        a.stats = stats.get();
      }
      ProfRegion pr(ctx, "knn_dr");
      const bool gen = a.k.nu_code == kNuGeneral;
      const int lr = m_v <= 32 ? 1 : (m_v <= 64 ? 2 : 4);
      auto dkern = lr == 1 ? (gen ? knn_dr_kernel<true, 1> : knn_dr_kernel<false, 1>)
                           : lr == 2 ? (gen ? knn_dr_kernel<true, 2> : knn_dr_kernel<false, 2>)
                                     : (gen ? knn_dr_kernel<true, 4> : knn_dr_kernel<false, 4>);
      const size_t dsmem = dr_smem(lr);
      STGP_CUDA(cudaFuncSetAttribute(dkern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsmem)));
      // ranks shard the queries by whole time buckets (contiguous rows), balanced by row count;
      // candidates (W, tiles) are replicated and the rows gathered afterwards
      int b0 = 0, b1 = nbucket;
      if (ctx->world > 1) {
        int r0 = 0, r1 = n;
        shard_rows(ctx, n, r0, r1);
        auto first_at = [&](int row) {
          return static_cast<int>(std::lower_bound(bstart.begin(), bstart.end() - 1, row) - bstart.begin());
        };
        b0 = ctx->rank == 0 ? 0 : first_at(r0);
        b1 = ctx->rank == ctx->world - 1 ? nbucket : first_at(r1);
      }
      a.tile0 = btile0[static_cast<size_t>(b0)];
      const int nt = btile0[static_cast<size_t>(b1)] - a.tile0;
      if (nt > 0) {
        dkern<<<nt, kDrThreads, dsmem, st>>>(a);
        launched(ctx);
      }
      gather_rows(ctx, nb->idx.get(), nb->dist.get(), n, m_v, bstart[static_cast<size_t>(b0)],
                  bstart[static_cast<size_t>(b1)]);
      lap("knn");
      if (a.stats) {
        unsigned long long h[64];
        STGP_CUDA(cudaMemcpyAsync(h, a.stats, 64 * 8, cudaMemcpyDeviceToHost, st));
        STGP_CUDA(cudaStreamSynchronize(st));
        std::fprintf(stderr,
                     "[stgp] d_r tiles (%d query tiles, %d groups): evaluated %llu pruned %llu; half filter skipped "
                     "%llu; with insertions: seed %llu, traversal %llu\n",
                     ntile, G, h[0], h[1], h[47], h[48], h[49]);
        for (int lg = 0; lg < 16; ++lg)
          std::fprintf(stderr, "[stgp]   lag %2d: evaluated %llu pruned %llu stops %llu\n", lg, h[2 + lg], h[18 + lg],
                       h[34 + lg]);
        const char* names[7] = {"tile selection", "live test",    "half filter", "exact Gram",
                                "d_r epilogue",   "merge",        "  of which fp16 Gram"};
        double tot = 0.0;
        for (int q = 0; q < 6; ++q) tot += static_cast<double>(h[50 + q]);
        for (int q = 0; q < 7; ++q)
          std::fprintf(stderr, "[stgp]   phase %-14s %6.1f%% of CTA cycles\n", names[q],
                       100.0 * static_cast<double>(h[50 + q]) / std::max(tot, 1.0));
      }
    }
    if (std::getenv("STGP_SPIN_SYNC")) {
      cudaError_t e;
      while ((e = cudaStreamQuery(st)) == cudaErrorNotReady) {
      }
      STGP_CUDA(e);
    } else {
      STGP_CUDA(cudaStreamSynchronize(st));
    }
    lap("sync");
    prof_collect(ctx);
    result = nb.release();
    lap("finish");
    frees_clk = std::chrono::steady_clock::now();
  }
  // (W, tiles and stats are released here, after the lap above)
  if (std::getenv("STGP_DR_HOSTLAPS"))
    std::fprintf(stderr, "[stgp] d_r phase %-12s %8.2f ms\n", "frees",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - frees_clk).count());
  return result;
}

}  // namespace stgp

extern "C" {

int stgp_residual_neighbors(stgp_dataset* ds, const stgp_params* theta, const stgp_inducing* ind, int m_v,
                            stgp_neighbors** out) {
  return guarded([&] {
    if (!ds || !theta || !ind || !out) config_error("stgp_residual_neighbors: null argument");
    Params p;
    std::memcpy(&p, theta, sizeof(p));
    validate_params(p);
    *out = spatial_search(ds, p, ind->xyt, m_v, STGP_METRIC_DR);
  });
}

}  // extern "C"

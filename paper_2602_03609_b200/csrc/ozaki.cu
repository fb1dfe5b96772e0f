// FP64 GEMM on the INT8 tensor cores (Ozaki scheme I, error-free slicing).
//
// B200's FP64 pipes (DMMA and DFMA) peak at ~37 TFLOP/s, while its int8 tensor cores run
// cuBLASLt IMMA at ~2.4 POPS (scripts/exp/imma_probe.py).  An FP64 product
//   C[r][j] = sum_c A[r][c] B[j][c]            (rows of A and B contiguous over c)
// is computed exactly up to the slicing truncation:
//   * row r of A is scaled by 2^-eA[r] into (-1, 1) and cut into S int8 slices of 7 bits each,
//     a = sum_s A_s 2^-7s (every step exact in FP64); B likewise per row j;
//   * the products A_s B_t with s + t = d share the scale 2^-7d and are one int8 GEMM over the
//     concatenated K = (d - 1) k (A slices stored consecutively, B slices in reverse order, so
//     each diagonal is a prefix of A's row times a suffix of B's row); its int32 result is exact
//     (|C_d| <= S k 127^2 < 2^31 for k < 2^31 / (S 127^2));
//   * C = 2^(eA + eB) sum_{d = 2}^{S + 1} 2^-7d C_d, summed in FP64 from the smallest term.
// Terms with s + t > S + 1 are dropped: the result carries ~7 S bits relative to
// max_c |A[r][c]| max_c |B[j][c]| k (S = 7: 49 bits; far below the 1e-8 parity tolerance of the
// evaluation, tests/test_gpu_ozaki.py measures it against cuBLAS DGEMM).
#include <cublasLt.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <memory>
#include <tuple>

#include "lowrank_common.cuh"
#include "ozaki.cuh"

namespace stgp {

namespace {

void lt_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS)
    throw Error(kInternal, std::string("cuBLASLt error in ") + what + ": " + std::to_string(static_cast<int>(s)));
}

// One warp per row: exponent of the row maximum (scale[r] = 2^e > max |row|), then the S slices
// (char4 stores).  reverse: slice t stored at (S - t) kp (B operand), else at (t - 1) kp.
__global__ void __launch_bounds__(256) slice_rows_kernel(long long nrows, int k, int kp, const double* __restrict__ A,
                                                         int lda, int S, bool reverse, int8_t* __restrict__ out,
                                                         long long ldo, double* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long r = warp; r < nrows; r += nw) {
    const double* a = A + r * lda;
    double mx = 0.0;
    for (int c = lane; c < k; c += 32) mx = fmax(mx, fabs(a[c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (lane == 0) scale[r] = ldexp(1.0, e);
    const double inv = ldexp(1.0, -e);
    int8_t* o = out + r * ldo;
    for (int c4 = lane * 4; c4 < kp; c4 += 128) {  // kp: k padded to 16 (zero slices)
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = c4 + u < k ? a[c4 + u] * inv : 0.0;  // exact: power-of-two scale
      for (int s = 1; s <= S; ++s) {
        char4 q;
        signed char qq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double w = v[u] * 128.0;  // exact
          const double t = trunc(w);      // |t| <= 127
          v[u] = w - t;                   // exact remainder in (-1, 1)
          qq[u] = static_cast<signed char>(t);
        }
        q.x = qq[0];
        q.y = qq[1];
        q.z = qq[2];
        q.w = qq[3];
        *reinterpret_cast<char4*>(o + (reverse ? (S - s) : (s - 1)) * kp + c4) = q;
      }
    }
  }
}

// Column form: A is m x n column-major (lda), optionally with column r divided by sqrt(colD[r]);
// the product runs over n in chunks of L.  Row j of
// chunk c is scaled by scale[c * m + j] = 2^e (> max over the chunk) and sliced into
// out[((c * m + j) * S + s - 1) * L + rl] and/or out_rev[((c * m + j) * S + S - s) * L + rl],
// through a shared-memory transpose of 32 rows x 128 columns so that both the loads and the int8
// stores are coalesced.
constexpr int kSlTileR = 128;
__global__ void __launch_bounds__(256) slice_cols_kernel(int m, long long n, int L, const double* __restrict__ A,
                                                         int lda, const double* __restrict__ colD, int S,
                                                         int8_t* __restrict__ out, int8_t* __restrict__ out_rev,
                                                         double* __restrict__ scale) {
  __shared__ double T[32][kSlTileR + 1];
  __shared__ double red[8][32];
  __shared__ double sinv[32];
  const int c = blockIdx.x, j0 = blockIdx.y * 32;
  const long long r0 = static_cast<long long>(c) * L, r1 = min(n, r0 + L);
  const int jj = threadIdx.x & 31, rr = threadIdx.x >> 5;
  const int j = j0 + jj;
  // column r of A enters as A(:, r) / sqrt(colD[r]) when colD is given (V' D^{-1/2} of the K product)
  auto val = [&](long long r) {
    const double a = A[r * lda + j];
    return colD ? a * __ldg(&colD[r]) : a;  // colD holds the factors 1 / sqrt(D_r) (rsqrt_vec_kernel)
  };
  double mx = 0.0;
  if (j < m) {
#pragma unroll 4
    for (long long r = r0 + rr; r < r1; r += 8) mx = fmax(mx, fabs(val(r)));
  }
  red[rr][jj] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = 0.0;
    for (int q = 0; q < 8; ++q) v = fmax(v, red[q][threadIdx.x]);
    int e = 0;
    if (v > 0.0) frexp(v, &e);
    sinv[threadIdx.x] = ldexp(1.0, -e);
    if (j0 + threadIdx.x < m) scale[static_cast<size_t>(c) * m + j0 + threadIdx.x] = ldexp(1.0, e);
  }
  __syncthreads();
  const int wj = threadIdx.x >> 3, wr = (threadIdx.x & 7) * 16;  // slicing: row wj, 16 columns
  for (long long t0 = r0; t0 < r0 + L; t0 += kSlTileR) {
    for (int q = rr; q < kSlTileR; q += 8) {
      const long long r = t0 + q;
      T[jj][q] = (j < m && r < r1) ? val(r) * sinv[jj] : 0.0;
    }
    __syncthreads();
    if (j0 + wj < m) {
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = T[wj][wr + u];
      const size_t base = (static_cast<size_t>(c) * m + j0 + wj) * S * static_cast<size_t>(L) + (t0 - r0) + wr;
      for (int s = 1; s <= S; ++s) {
        alignas(16) signed char qq[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double w = v[u] * 128.0;
          const double tq = trunc(w);
          v[u] = w - tq;
          qq[u] = static_cast<signed char>(tq);
        }
        const int4 q = *reinterpret_cast<const int4*>(qq);
        if (out) *reinterpret_cast<int4*>(out + base + static_cast<size_t>(s - 1) * L) = q;
        if (out_rev) *reinterpret_cast<int4*>(out_rev + base + static_cast<size_t>(S - s) * L) = q;
      }
    }
    __syncthreads();
  }
}

// C[r * ldc + j] = sA[r] sB[j] sum_{d = S+1 .. 2} 2^-7d Cd[d][r * mp + j]   (one row per iteration,
// 4 consecutive j per thread: m, mp and ldc are multiples of 4, rows 16-byte aligned)
__global__ void __launch_bounds__(256) combine_rows_kernel(long long nrows, int m, int mp, const int32_t* __restrict__ Cd,
                                                           long long dstride, int S, const double* __restrict__ sA,
                                                           const double* __restrict__ sB, double* __restrict__ C,
                                                           int ldc) {
  for (long long r = blockIdx.x; r < nrows; r += gridDim.x) {
    const double fa = sA[r];
    const int32_t* src = Cd + r * mp;
    for (int j = threadIdx.x * 4; j < m; j += blockDim.x * 4) {
      int4 v[12];
#pragma unroll
      for (int d = 0; d < 12; ++d)
        if (d < S) v[d] = __ldg(reinterpret_cast<const int4*>(src + d * dstride + j));
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, w = ldexp(1.0, -7 * (S + 1));  // smallest diagonal first
#pragma unroll
      for (int d = 11; d >= 0; --d)
        if (d < S) {  // exact products (power-of-two weights), one rounding per add
          a0 = fma(static_cast<double>(v[d].x), w, a0);
          a1 = fma(static_cast<double>(v[d].y), w, a1);
          a2 = fma(static_cast<double>(v[d].z), w, a2);
          a3 = fma(static_cast<double>(v[d].w), w, a3);
          w *= 128.0;
        }
      double* o = C + r * ldc + j;
      const double4 fb = *reinterpret_cast<const double4*>(sB + j);
      *reinterpret_cast<double2*>(o) = make_double2(a0 * fa * fb.x, a1 * fa * fb.y);
      *reinterpret_cast<double2*>(o + 2) = make_double2(a2 * fa * fb.z, a3 * fa * fb.w);
    }
  }
}

__global__ void rsqrt_vec_kernel(long long n, const double* __restrict__ d, double* __restrict__ f) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    f[i] = 1.0 / sqrt(d[i]);  // the factor of lowrank.cu scale_cols_kernel
}

// C[j * ldc + i] = sum_c sA[c m + j] sB[c m + i] sum_d 2^-7d Cd[d][c][j * mp + i]   (chunks in order)
__global__ void __launch_bounds__(256) combine_cols_kernel(int m, int mp, int nch, const int32_t* __restrict__ Cd,
                                                           long long dstride, long long cstride, int S,
                                                           const double* __restrict__ sA,
                                                           const double* __restrict__ sB, double* __restrict__ C,
                                                           int ldc) {
  const long long total = static_cast<long long>(m) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e / m), i = static_cast<int>(e - static_cast<long long>(j) * m);
    double out = 0.0;
    for (int c = 0; c < nch; ++c) {
      const int32_t* src = Cd + c * cstride + static_cast<long long>(j) * mp + i;
      double acc = 0.0, w = ldexp(1.0, -7 * (S + 1));
      for (int d = S - 1; d >= 0; --d) {
        acc = fma(static_cast<double>(src[d * dstride]), w, acc);
        w *= 128.0;
      }
      out = fma(acc, sA[static_cast<size_t>(c) * m + j] * sB[static_cast<size_t>(c) * m + i], out);
    }
    C[static_cast<long long>(j) * ldc + i] = out;
  }
}

struct LtPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulAlgo_t algo{};
  ~LtPlan() {
    if (la) cublasLtMatrixLayoutDestroy(la);
    if (lb) cublasLtMatrixLayoutDestroy(lb);
    if (lc) cublasLtMatrixLayoutDestroy(lc);
    if (op) cublasLtMatmulDescDestroy(op);
  }
};

}  // namespace

struct OzakiState {
  cublasLtHandle_t lt = nullptr;
  DevBuf<unsigned char> ws;
  DevBuf<int8_t> As, Bs;
  DevBuf<int32_t> Cd;
  DevBuf<double> sA, sB, colf;
  std::map<std::tuple<int, int, long long, int, int, int>, std::unique_ptr<LtPlan>> plans;
  ~OzakiState() {
    plans.clear();
    if (lt) cublasLtDestroy(lt);
  }
};

void ozaki_release(stgp_ctx* ctx) {
  delete ctx->ozaki;
  ctx->ozaki = nullptr;
}

int ozaki_slices() {
  static const int s = [] {
    const char* e = std::getenv("STGP_OZAKI_S");
    return std::max(2, std::min(12, e ? std::atoi(e) : 7));
  }();
  return s;
}

bool ozaki_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STGP_OZAKI");  // A/B switch: 0 = cuBLAS DGEMM
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

static OzakiState* state(stgp_ctx* ctx) {
  if (!ctx->ozaki) {
    ctx->ozaki = new OzakiState();
    lt_check(cublasLtCreate(&ctx->ozaki->lt), "create");
    ctx->ozaki->ws.alloc(64ull << 20);
  }
  return ctx->ozaki;
}

// Plan for Cd (m x ncols, int32, ld mp) = op(Bseg)^T (m x K) * Aseg (K x ncols), both K-contiguous
// with leading dimension ldk (TN int8 IMMA); `batch` products strided by bstride (operands) and
// cstride (results).
static LtPlan* plan_for(OzakiState* oz, int m, int mp, int K, long long ncols, int ldk, int batch = 1,
                        long long bstride = 0, long long cstride = 0) {
  auto key = std::make_tuple(m, K, ncols, ldk, mp, batch);
  auto it = oz->plans.find(key);
  if (it != oz->plans.end()) return it->second.get();
  auto p = std::make_unique<LtPlan>();
  lt_check(cublasLtMatmulDescCreate(&p->op, CUBLAS_COMPUTE_32I, CUDA_R_32I), "desc");
  const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  lt_check(cublasLtMatmulDescSetAttribute(p->op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)), "transa");
  lt_check(cublasLtMatmulDescSetAttribute(p->op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)), "transb");
  lt_check(cublasLtMatrixLayoutCreate(&p->la, CUDA_R_8I, K, m, ldk), "layout a");
  lt_check(cublasLtMatrixLayoutCreate(&p->lb, CUDA_R_8I, K, ncols, ldk), "layout b");
  lt_check(cublasLtMatrixLayoutCreate(&p->lc, CUDA_R_32I, m, ncols, mp), "layout c");
  if (batch > 1) {
    for (auto* l : {p->la, p->lb}) {
      lt_check(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof(batch)), "batch");
      lt_check(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &bstride,
                                                sizeof(bstride)), "bstride");
    }
    lt_check(cublasLtMatrixLayoutSetAttribute(p->lc, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof(batch)), "batch");
    lt_check(cublasLtMatrixLayoutSetAttribute(p->lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &cstride,
                                              sizeof(cstride)), "cstride");
  }
  cublasLtMatmulPreference_t pref;
  lt_check(cublasLtMatmulPreferenceCreate(&pref), "pref");
  const size_t wsz = oz->ws.n;
  lt_check(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz)),
           "pref ws");
  cublasLtMatmulHeuristicResult_t res{};
  int found = 0;
  lt_check(cublasLtMatmulAlgoGetHeuristic(oz->lt, p->op, p->la, p->lb, p->lc, p->lc, pref, 1, &res, &found),
           "heuristic");
  cublasLtMatmulPreferenceDestroy(pref);
  if (found < 1) throw Error(kInternal, "cuBLASLt: no int8 IMMA algorithm for the Ozaki slices");
  p->algo = res.algo;
  LtPlan* raw = p.get();
  oz->plans[key] = std::move(p);
  return raw;
}

static void lt_matmul(stgp_ctx* ctx, OzakiState* oz, LtPlan* p, const int8_t* a, const int8_t* b, int32_t* c) {
  const int32_t one = 1, zero = 0;
  lt_check(cublasLtMatmul(oz->lt, p->op, &one, a, p->la, b, p->lb, &zero, c, p->lc, c, p->lc, &p->algo, oz->ws.get(),
                          oz->ws.n, ctx->stream),
           "matmul");
  launched(ctx);
}

void ozaki_gemm_rows(stgp_ctx* ctx, long long n, int m, int k, const double* A, int lda, const double* B, int ldb,
                     double* C, int ldc) {
  if (n <= 0 || m <= 0) return;
  if (m % 4 || ldc % 4) config_error("ozaki_gemm_rows: m and ldc must be multiples of 4");
  const int S = ozaki_slices();
  const int kp = (k + 15) / 16 * 16;  // slice stride: every diagonal segment 16-byte aligned
  if (static_cast<long long>(S) * kp * 127 * 127 >= (1LL << 31)) config_error("ozaki: k too large for exact int32");
  OzakiState* oz = state(ctx);
  cudaStream_t st = ctx->stream;
  const int ldk = S * kp;
  const int mp = (m + 3) / 4 * 4;  // int32 result rows (16-byte aligned columns)
  // B slices (m rows, reversed slice order) and scales
  oz->Bs.ensure(static_cast<size_t>(m) * ldk);
  oz->sB.ensure(m);
  slice_rows_kernel<<<grid_for(static_cast<long long>(m) * 32, 256), 256, 0, st>>>(m, k, kp, B, ldb, S, true,
                                                                                 oz->Bs.get(), ldk, oz->sB.get());
  launched(ctx);
  const long long chunk = std::min<long long>(n, std::max<long long>(16384, (1LL << 28) / mp));  // Cd ~ S GB
  oz->As.ensure(static_cast<size_t>(chunk) * ldk);
  oz->sA.ensure(static_cast<size_t>(chunk));
  const long long dstride = chunk * mp;
  oz->Cd.ensure(static_cast<size_t>(S) * dstride);
  for (long long r0 = 0; r0 < n; r0 += chunk) {
    const long long nr = std::min(chunk, n - r0);
    slice_rows_kernel<<<grid_for(nr * 32, 256), 256, 0, st>>>(nr, k, kp, A + r0 * lda, lda, S, false, oz->As.get(),
                                                              ldk, oz->sA.get());
    launched(ctx);
    for (int d = 2; d <= S + 1; ++d) {
      LtPlan* p = plan_for(oz, m, mp, (d - 1) * kp, nr, ldk);
      lt_matmul(ctx, oz, p, oz->Bs.get() + static_cast<size_t>(S - d + 1) * kp, oz->As.get(),
                oz->Cd.get() + (d - 2) * dstride);
    }
    combine_rows_kernel<<<static_cast<int>(std::min<long long>(nr, ctx->num_sms * 16)), 256, 0, st>>>(
        nr, m, mp, oz->Cd.get(), dstride, S, oz->sA.get(), oz->sB.get(), C + r0 * ldc, ldc);
    launched(ctx);
  }
}

void ozaki_gemm_cols(stgp_ctx* ctx, int m, long long n, const double* A, int lda, const double* B, int ldb, double* C,
                     int ldc, const double* colD) {
  if (m <= 0) return;
  const int S = ozaki_slices();
  OzakiState* oz = state(ctx);
  cudaStream_t st = ctx->stream;
  // chunk of the reduction: exact int32 for the longest diagonal, (S) L 127^2 < 2^31
  const long long lmax = ((1LL << 31) - 1) / (static_cast<long long>(S) * 127 * 127);
  const int L = static_cast<int>(std::min<long long>(lmax / kSlTileR * kSlTileR, (n + kSlTileR - 1) / kSlTileR * kSlTileR));
  const int nch = static_cast<int>((n + L - 1) / L);
  const int mp = (m + 3) / 4 * 4;
  const long long ldk = static_cast<long long>(S) * L;
  const long long bstride = static_cast<long long>(m) * ldk;
  const size_t sl = static_cast<size_t>(nch) * bstride;
  oz->As.ensure(sl);
  oz->sA.ensure(static_cast<size_t>(nch) * m);
  const bool same = A == B && lda == ldb;  // A A^T: one pass writes both slice orders
  if (colD) {
    oz->colf.ensure(static_cast<size_t>(n));
    rsqrt_vec_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, colD, oz->colf.get());
    launched(ctx);
    colD = oz->colf.get();
  }
  oz->Bs.ensure(sl);
  oz->sB.ensure(static_cast<size_t>(nch) * m);
  const dim3 grid(nch, (m + 31) / 32);
  slice_cols_kernel<<<grid, 256, 0, st>>>(m, n, L, A, lda, colD, S, oz->As.get(), same ? oz->Bs.get() : nullptr,
                                          oz->sA.get());
  launched(ctx);
  if (!same) {
    slice_cols_kernel<<<grid, 256, 0, st>>>(m, n, L, B, ldb, colD, S, nullptr, oz->Bs.get(), oz->sB.get());
    launched(ctx);
  }
  const double* sB = same ? oz->sA.get() : oz->sB.get();
  const long long cstride = static_cast<long long>(m) * mp;
  const long long dstride = nch * cstride;
  oz->Cd.ensure(static_cast<size_t>(S) * dstride);
  for (int d = 2; d <= S + 1; ++d) {
    LtPlan* p = plan_for(oz, m, mp, (d - 1) * L, m, static_cast<int>(ldk), nch, bstride, cstride);
    lt_matmul(ctx, oz, p, oz->Bs.get() + static_cast<size_t>(S - d + 1) * L, oz->As.get(),
              oz->Cd.get() + (d - 2) * dstride);
  }
  combine_cols_kernel<<<grid_for(static_cast<long long>(m) * m, 256), 256, 0, st>>>(
      m, mp, nch, oz->Cd.get(), dstride, cstride, S, oz->sA.get(), sB, C, ldc);
  launched(ctx);
}

}  // namespace stgp

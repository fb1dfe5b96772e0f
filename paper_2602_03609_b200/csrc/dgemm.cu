// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) GEMM for the dense low-rank algebra: the n x M^2
// triangular products (W = L_m^{-1} U, omega = L_m^{-T} omega'), the M x M x n Gram products of the
// DMMA path (M < 512), the M x M pieces of the Woodbury cores and the blocked Cholesky / triangular
// solves of dense.cu.  Column-major operands, C = alpha op(A) op(B) + beta C.
//
// CTA tile 64 x 128, K step 16, three cp.async stages (25.6 KB each), four warps of 32 x 64 (4 x 8 DMMA
// tiles, 64 accumulator registers).  Shared tiles are stored k-major with a row pitch of 4 mod 16 doubles
// so the fragment loads of a half-warp hit distinct banks.  Triangular A (explicit inverse factors,
// zero outside the triangle) restricts each row block's K range to the triangle's support, which gives
// TRMM its n M^2 / 2 cost.  Long reductions (K ~ n, small C) split K over grid.z into partial tiles that
// a second kernel sums in split order (deterministic).
#include <algorithm>

#include "dense.cuh"
#include "engine.hpp"

namespace stgp {
namespace {

constexpr int kGM = 64, kGN = 128, kGK = 16, kGStages = 3, kGThreads = 128;
constexpr int kPA = kGM + 4, kPB = kGN + 4;  // shared pitches (doubles), 4 mod 16
constexpr int kStageD = kGK * (kPA + kPB);   // doubles per stage
constexpr int kGSmem = kGStages * kStageD * 8;

__device__ __forceinline__ void cp8(double* dst, const double* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(valid ? src : nullptr),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct GemmArgs {
  int m, n;
  long long k;
  const double* A;
  long long lda;
  const double* B;
  long long ldb;
  double* C;  // split == 1: C = alpha acc + beta C; else partial P[z] (ldc) = acc
  long long ldc;
  double alpha, beta;
  int tri;       // 0: none; 1: op(A) lower (row i sums k <= i); 2: op(A) upper (k >= i)
  int splits;
  long long pstride;
};

// stage the (k0 .. k0+15) slice of op(A) (rows m0..m0+63) and op(B) (cols n0..n0+127)
template <bool TA, bool TB>
__device__ __forceinline__ void load_stage(const GemmArgs& g, double* sA, double* sB, int m0, int n0, long long k0) {
  const int t = threadIdx.x;
#pragma unroll
  for (int i = 0; i < kGM * kGK / kGThreads; ++i) {
    int mm, kk;
    if (!TA) {  // A col-major m x k: contiguous along m
      const int e = t + i * kGThreads;
      mm = e % kGM;
      kk = e / kGM;
    } else {  // op(A) = A^T, A is k x m: contiguous along k
      const int e = t + i * kGThreads;
      kk = e % kGK;
      mm = e / kGK;
    }
    const int gm = m0 + mm;
    const long long gk = k0 + kk;
    const bool ok = gm < g.m && gk < g.k;
    const double* src = TA ? g.A + gk + static_cast<long long>(gm) * g.lda : g.A + gm + gk * g.lda;
    cp8(sA + kk * kPA + mm, src, ok);
  }
#pragma unroll
  for (int i = 0; i < kGN * kGK / kGThreads; ++i) {
    int nn, kk;
    if (!TB) {  // B col-major k x n: contiguous along k
      const int e = t + i * kGThreads;
      kk = e % kGK;
      nn = e / kGK;
    } else {  // op(B) = B^T, B is n x k: contiguous along n
      const int e = t + i * kGThreads;
      nn = e % kGN;
      kk = e / kGN;
    }
    const int gn = n0 + nn;
    const long long gk = k0 + kk;
    const bool ok = gn < g.n && gk < g.k;
    const double* src = TB ? g.B + gn + gk * g.ldb : g.B + gk + static_cast<long long>(gn) * g.ldb;
    cp8(sB + kk * kPB + nn, src, ok);
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(kGThreads) dgemm_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double gsm[];
  const int m0 = blockIdx.y * kGM, n0 = blockIdx.x * kGN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 64;
  const int gq = lane & 3, gg = lane >> 2;
  // K range: triangle support, then this split's share (whole K steps)
  long long kb = 0, ke = g.k;
  if (g.tri == 1) ke = std::min<long long>(g.k, m0 + kGM);
  if (g.tri == 2) kb = (m0 / kGK) * kGK;
  const long long nsteps = (ke - kb + kGK - 1) / kGK;
  const long long s0 = nsteps * blockIdx.z / g.splits, s1 = nsteps * (blockIdx.z + 1) / g.splits;
  const long long steps = s1 - s0;
  double acc[4][8][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // prologue
#pragma unroll
  for (int s = 0; s < kGStages - 1; ++s) {
    if (s < steps) load_stage<TA, TB>(g, gsm + s * kStageD, gsm + s * kStageD + kGK * kPA, m0, n0, kb + (s0 + s) * kGK);
    cp_commit();
  }
  for (long long it = 0; it < steps; ++it) {
    cp_wait<kGStages - 2>();
    __syncthreads();
    {  // prefetch the step kGStages - 1 ahead into the slot freed by the previous iteration
      const long long nx = it + kGStages - 1;
      const int slot = static_cast<int>(nx % kGStages);
      if (nx < steps)
        load_stage<TA, TB>(g, gsm + slot * kStageD, gsm + slot * kStageD + kGK * kPA, m0, n0, kb + (s0 + nx) * kGK);
      cp_commit();
    }
    const double* sA = gsm + static_cast<int>(it % kGStages) * kStageD;
    const double* sB = sA + kGK * kPA;
#pragma unroll
    for (int kk = 0; kk < kGK; kk += 4) {
      double a[4], b[8];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sA[(kk + gq) * kPA + wm + mi * 8 + gg];
#pragma unroll
      for (int ni = 0; ni < 8; ++ni) b[ni] = sB[(kk + gq) * kPB + wn + ni * 8 + gg];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  }
  cp_wait<0>();
  // epilogue: thread holds C[wm + mi 8 + gg][wn + ni 8 + 2 gq + {0, 1}]
  double* C = g.splits > 1 ? g.C + blockIdx.z * g.pstride : g.C;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int r = m0 + wm + mi * 8 + gg;
    if (r >= g.m) continue;
#pragma unroll
    for (int ni = 0; ni < 8; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + ni * 8 + 2 * gq + h;
        if (c >= g.n) continue;
        double* o = C + r + static_cast<long long>(c) * g.ldc;
        if (g.splits > 1) *o = acc[mi][ni][h];
        else *o = g.beta == 0.0 ? g.alpha * acc[mi][ni][h] : fma(g.alpha, acc[mi][ni][h], g.beta * *o);
      }
  }
}

// C = alpha sum_z P_z + beta C, in split order
__global__ void splitk_reduce_kernel(int m, int n, int splits, const double* __restrict__ P, long long ldp,
                                     long long pstride, double alpha, double beta, double* __restrict__ C, long long ldc) {
  const long long total = static_cast<long long>(m) * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = e / m, r = e - c * m;
    double s = P[r + c * ldp];
    for (int z = 1; z < splits; ++z) s += P[z * pstride + r + c * ldp];
    double* o = C + r + c * ldc;
    *o = beta == 0.0 ? alpha * s : fma(alpha, s, beta * *o);
  }
}

template <bool TA, bool TB>
void launch_gemm(stgp_ctx* ctx, const GemmArgs& g, dim3 grid) {
  static bool attr = false;
  if (!attr) {
    STGP_CUDA(cudaFuncSetAttribute(dgemm_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kGSmem));
    attr = true;
  }
  dgemm_kernel<TA, TB><<<grid, kGThreads, kGSmem, ctx->stream>>>(g);
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
}

}  // namespace

void dev_gemm_tri(stgp_ctx* ctx, bool ta, bool tb, int m, int n, long long k, double alpha, const double* A,
                  long long lda, const double* B, long long ldb, double beta, double* C, long long ldc, int tri) {
  if (m <= 0 || n <= 0) return;
  if (k <= 0) {  // C = beta C
    GemmArgs z{m, n, 0, A, lda, B, ldb, C, ldc, alpha, beta, 0, 1, 0};
    dim3 grid((n + kGN - 1) / kGN, (m + kGM - 1) / kGM, 1);
    launch_gemm<false, false>(ctx, z, grid);
    return;
  }
  const long long tiles = static_cast<long long>((n + kGN - 1) / kGN) * ((m + kGM - 1) / kGM);
  // split a long reduction until the grid covers ~2 waves of CTAs (3 resident per SM)
  int splits = 1;
  const long long want = 2LL * 3 * ctx->num_sms;
  if (tiles < want && tri == 0) {
    const long long ksteps = (k + kGK - 1) / kGK;
    splits = static_cast<int>(std::min<long long>({(want + tiles - 1) / tiles, ksteps / 32, 64LL}));
    splits = std::max(splits, 1);
  }
  GemmArgs g{m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, tri, splits, 0};
  DevBuf<double>* part = nullptr;
  if (splits > 1) {
    part = &ctx->gemm_part;
    g.ldc = m;
    g.pstride = static_cast<long long>(m) * n;
    part->ensure(static_cast<size_t>(splits) * g.pstride);
    g.C = part->get();
  }
  // grid.x over n (up to 2^31 - 1 tiles), grid.y over m, grid.z over the K splits
  const dim3 grid(static_cast<unsigned>((n + kGN - 1) / kGN), (m + kGM - 1) / kGM, splits);
  if (!ta && !tb) launch_gemm<false, false>(ctx, g, grid);
  else if (!ta && tb) launch_gemm<false, true>(ctx, g, grid);
  else if (ta && !tb) launch_gemm<true, false>(ctx, g, grid);
  else launch_gemm<true, true>(ctx, g, grid);
  if (splits > 1) {
    const long long total = static_cast<long long>(m) * n;
    splitk_reduce_kernel<<<static_cast<int>(std::min<long long>((total + 255) / 256, ctx->num_sms * 16LL)), 256, 0,
                           ctx->stream>>>(m, n, splits, part->get(), m, g.pstride, alpha, beta, C, ldc);
    ++ctx->launches;
    STGP_LAUNCH_CHECK();
  }
}

}  // namespace stgp

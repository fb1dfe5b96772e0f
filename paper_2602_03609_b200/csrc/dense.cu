#include <climits>
#include <string>

#include "dense.cuh"
#include "engine.hpp"

namespace stgp {

void cublas_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) throw Error(kInternal, std::string("cuBLAS ") + what + " failed: " + std::to_string(s));
}

namespace {

constexpr int kNB = 64;

// Factor one diagonal block (nb <= 64) in place with one CTA; flags[0] = 1 on a
// non-positive pivot.  Right-looking, column by column.
__global__ void potrf_diag_kernel(double* A, int ld, int j0, int nb, int* flag) {
  __shared__ double s[kNB][kNB + 1];
  const int tid = threadIdx.x;
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int r = e % nb, c = e / nb;
    s[r][c] = A[static_cast<size_t>(j0 + c) * ld + j0 + r];
  }
  __syncthreads();
  __shared__ int bad;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (tid == 0) {
      const double p = s[j][j];
      if (!(p > 0.0)) bad = 1;
      s[j][j] = sqrt(p);
    }
    __syncthreads();
    if (bad) break;
    const double d = s[j][j];
    for (int r = j + 1 + tid; r < nb; r += blockDim.x) s[r][j] /= d;
    __syncthreads();
    for (int e = tid; e < (nb - j - 1) * (nb - j - 1); e += blockDim.x) {
      const int r = j + 1 + e % (nb - j - 1), c = j + 1 + e / (nb - j - 1);
      if (c <= r) s[r][c] = fma(-s[r][j], s[c][j], s[r][c]);
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) *flag = 1;
    return;
  }
  for (int e = tid; e < nb * nb; e += blockDim.x) {
    const int r = e % nb, c = e / nb;
    if (c <= r) A[static_cast<size_t>(j0 + c) * ld + j0 + r] = s[r][c];
  }
}

__global__ void logdiag_kernel(const double* L, int ld, int n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += log(L[static_cast<size_t>(i) * ld + i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = 2.0 * red[0];
}

__global__ void symmetrize_kernel(double* A, int ld, int n) {
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < static_cast<long long>(n) * n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e % n), c = static_cast<int>(e / n);
    if (r < c) A[static_cast<size_t>(c) * ld + r] = A[static_cast<size_t>(r) * ld + c];
  }
}

}  // namespace

bool dev_cholesky(stgp_ctx* ctx, double* A, int ld, int n) {
  DevBuf<int>& flag = ctx->iscr;
  flag.ensure(1);
  STGP_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), ctx->stream));
  const double one = 1.0, mone = -1.0;
  for (int j0 = 0; j0 < n; j0 += kNB) {
    const int nb = std::min(kNB, n - j0);
    potrf_diag_kernel<<<1, 256, 0, ctx->stream>>>(A, ld, j0, nb, flag.get());
    ++ctx->launches;
    STGP_LAUNCH_CHECK();
    const int rest = n - j0 - nb;
    if (rest > 0) {
      // A21 <- A21 L11^{-T}
      cublas_check(cublasDtrsm(ctx->cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T,
                               CUBLAS_DIAG_NON_UNIT, rest, nb, &one, A + static_cast<size_t>(j0) * ld + j0, ld,
                               A + static_cast<size_t>(j0) * ld + j0 + nb, ld),
                   "trsm(potrf)");
      // A22 <- A22 - A21 A21^T
      cublas_check(cublasDsyrk(ctx->cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, rest, nb, &mone,
                               A + static_cast<size_t>(j0) * ld + j0 + nb, ld, &one,
                               A + static_cast<size_t>(j0 + nb) * ld + j0 + nb, ld),
                   "syrk(potrf)");
    }
  }
  int h = 0;
  flag.download(&h, 1, ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  return h == 0;
}

double dev_logdet_chol(stgp_ctx* ctx, const double* L, int ld, int n) {
  DevBuf<double>& out = ctx->dscr;
  out.ensure(1);
  logdiag_kernel<<<1, 256, 0, ctx->stream>>>(L, ld, n, out.get());
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
  double h = 0.0;
  out.download(&h, 1, ctx->stream);
  STGP_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

void dev_trsm_left(stgp_ctx* ctx, const double* L, int ldl, int n, double* B, int ldb, long long ncols, bool transpose) {
  const double one = 1.0;
  const long long chunk = std::max<long long>(1, ((1LL << 31) - 1) / ldb);  // < 2^31 elements per call
  for (long long c0 = 0; c0 < ncols; c0 += chunk) {
    const int nc = static_cast<int>(std::min(chunk, ncols - c0));
    cublas_check(cublasDtrsm(ctx->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, transpose ? CUBLAS_OP_T : CUBLAS_OP_N,
                             CUBLAS_DIAG_NON_UNIT, n, nc, &one, L, ldl, B + static_cast<size_t>(c0) * ldb, ldb),
                 "trsm");
  }
}

static __global__ void identity_kernel(double* A, int ld, int n) {
  const long long total = static_cast<long long>(ld) * n;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    A[e] = (e % ld == e / ld) ? 1.0 : 0.0;
}

void dev_tri_inverse(stgp_ctx* ctx, const double* L, int ld, int n, double* Linv) {
  const long long total = static_cast<long long>(ld) * n;
  identity_kernel<<<static_cast<int>(std::min<long long>((total + 255) / 256, 4096)), 256, 0, ctx->stream>>>(Linv, ld, n);
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
  dev_trsm_left(ctx, L, ld, n, Linv, ld, n, false);
}

void dev_trmm_left(stgp_ctx* ctx, const double* T, int ldt, int n, const double* B, int ldb, long long ncols,
                   bool transpose, double* C, int ldc) {
  const double one = 1.0;
  const long long chunk = std::max<long long>(1, ((1LL << 31) - 1) / std::max(ldb, ldc));  // < 2^31 elements per call
  for (long long c0 = 0; c0 < ncols; c0 += chunk) {
    const int nc = static_cast<int>(std::min(chunk, ncols - c0));
    cublas_check(cublasDtrmm(ctx->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, transpose ? CUBLAS_OP_T : CUBLAS_OP_N,
                             CUBLAS_DIAG_NON_UNIT, n, nc, &one, T, ldt, B + static_cast<size_t>(c0) * ldb, ldb,
                             C + static_cast<size_t>(c0) * ldc, ldc),
                 "trmm");
  }
}

void dev_syrk(stgp_ctx* ctx, int n, long long k, double alpha, const double* A, int lda, double beta, double* C,
              int ldc) {
  cublas_check(cublasDsyrk(ctx->cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, n, static_cast<int>(k), &alpha, A, lda,
                           &beta, C, ldc),
               "syrk");
}

void dev_gemm(stgp_ctx* ctx, bool ta, bool tb, int m, int n, long long k, double alpha, const double* A, int lda,
              const double* B, int ldb, double beta, double* C, int ldc) {
  cublas_check(cublasDgemm(ctx->cublas, ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb ? CUBLAS_OP_T : CUBLAS_OP_N, m, n,
                           static_cast<int>(k), &alpha, A, lda, B, ldb, &beta, C, ldc),
               "gemm");
}

// C = alpha A A^T (n x n, both triangles) as GEMMs on the lower blocks of an nb x nb partition:
// (nb + 1) / (2 nb) of the full product's flops at GEMM efficiency (cuBLAS SYRK tiles this
// small-output / long-K shape poorly).  Block edges are multiples of 16.
void dev_syrk_blocked(stgp_ctx* ctx, int n, long long k, double alpha, const double* A, int lda, double* C, int ldc,
                      int nb) {
  nb = std::max(1, std::min(nb, (n + 15) / 16));
  const int bs = ((n + nb - 1) / nb + 15) / 16 * 16;
  for (int i0 = 0; i0 < n; i0 += bs)
    for (int j0 = 0; j0 <= i0; j0 += bs) {
      const int mi = std::min(bs, n - i0), mj = std::min(bs, n - j0);
      dev_gemm(ctx, false, true, mi, mj, k, alpha, A + i0, lda, A + j0, lda, 0.0, C + static_cast<size_t>(j0) * ldc + i0,
               ldc);
    }
  dev_symmetrize_lower(ctx, C, ldc, n);
}

// C = alpha A B^T for a product known to be symmetric (e.g. W diag(phi) W^T with B = W diag(phi)):
// GEMMs on the lower blocks of an nb x nb partition, mirrored.
void dev_gemm_sym_blocked(stgp_ctx* ctx, int n, long long k, double alpha, const double* A, int lda, const double* B,
                          int ldb, double* C, int ldc, int nb) {
  nb = std::max(1, std::min(nb, (n + 15) / 16));
  const int bs = ((n + nb - 1) / nb + 15) / 16 * 16;
  for (int i0 = 0; i0 < n; i0 += bs)
    for (int j0 = 0; j0 <= i0; j0 += bs) {
      const int mi = std::min(bs, n - i0), mj = std::min(bs, n - j0);
      dev_gemm(ctx, false, true, mi, mj, k, alpha, A + i0, lda, B + j0, ldb, 0.0, C + static_cast<size_t>(j0) * ldc + i0,
               ldc);
    }
  dev_symmetrize_lower(ctx, C, ldc, n);
}

void dev_gemv(stgp_ctx* ctx, bool ta, int m, long long n, double alpha, const double* A, int lda, const double* x,
              double beta, double* y) {
  cublas_check(cublasDgemv(ctx->cublas, ta ? CUBLAS_OP_T : CUBLAS_OP_N, m, static_cast<int>(n), &alpha, A, lda, x, 1,
                           &beta, y, 1),
               "gemv");
}

void dev_symmetrize_lower(stgp_ctx* ctx, double* A, int ld, int n) {
  const long long total = static_cast<long long>(n) * n;
  symmetrize_kernel<<<static_cast<int>(std::min<long long>((total + 255) / 256, 4096)), 256, 0, ctx->stream>>>(A, ld, n);
  ++ctx->launches;
  STGP_LAUNCH_CHECK();
}

}  // namespace stgp

// Dense FP64 linear algebra on the device for the M x M / M x n low-rank pieces, all on the repo's own
// kernels: the DMMA GEMM of dgemm.cu (TRMM with explicit triangular factors, SYRK as lower-block GEMMs,
// split-K long reductions), blocked triangular solves and a blocked Cholesky that reports failure
// instead of producing NaNs (Eigen's LLT info() semantics, used by the jitter ladders).
#pragma once

#include "common.cuh"

struct stgp_ctx;

namespace stgp {

// C = alpha op(A) op(B) + beta C (column-major, DMMA); tri: 0 general, 1 op(A) lower with a zero upper
// part (row i sums k <= i), 2 op(A) upper with a zero lower part (k >= i)
void dev_gemm_tri(stgp_ctx* ctx, bool ta, bool tb, int m, int n, long long k, double alpha, const double* A,
                  long long lda, const double* B, long long ldb, double beta, double* C, long long ldc, int tri);
// out = (L L^T)^{-1} from the Cholesky factor L (explicit, exactly symmetric)
void dev_chol_inverse(stgp_ctx* ctx, const double* L, int ld, int n, double* out);
// W <- Linv^T W Linv for an explicit lower-triangular Linv (zero upper part)
void dev_congruence_t(stgp_ctx* ctx, const double* Linv, int ld, int n, double* W);
// B (nrows x n, ldb) <- B L^{-1} for lower-triangular L
void dev_trsm_right(stgp_ctx* ctx, const double* L, int ldl, int n, double* B, int ldb, int nrows);

// In-place lower Cholesky of the leading n x n block of A (column-major, ld).
// Returns false when a pivot is not positive (the factor is then unusable).
bool dev_cholesky(stgp_ctx* ctx, double* A, int ld, int n);
// 2 * sum log diag(L)
double dev_logdet_chol(stgp_ctx* ctx, const double* L, int ld, int n);
// B <- op(L)^{-1} B for lower-triangular L (n x n), B n x ncols (ldb).
void dev_trsm_left(stgp_ctx* ctx, const double* L, int ldl, int n, double* B, int ldb, long long ncols,
                   bool transpose);
// Linv = L^{-1} (lower triangular, n x n, zero upper part); out-of-place
void dev_tri_inverse(stgp_ctx* ctx, const double* L, int ld, int n, double* Linv);
// C = op(T) B for lower-triangular T (n x n): out-of-place triangular multiply
void dev_trmm_left(stgp_ctx* ctx, const double* T, int ldt, int n, const double* B, int ldb, long long ncols,
                   bool transpose, double* C, int ldc);
// C (n x n, lower) = alpha * A A^T + beta * C, A n x k (lda)
void dev_syrk(stgp_ctx* ctx, int n, long long k, double alpha, const double* A, int lda, double beta, double* C,
              int ldc);
// C = alpha op(A) op(B) + beta C
void dev_gemm(stgp_ctx* ctx, bool ta, bool tb, int m, int n, long long k, double alpha, const double* A, int lda,
              const double* B, int ldb, double beta, double* C, int ldc);
// y = alpha op(A) x + beta y
void dev_gemv(stgp_ctx* ctx, bool ta, int m, long long n, double alpha, const double* A, int lda, const double* x,
              double beta, double* y);
// copy the lower triangle into the upper triangle
void dev_symmetrize_lower(stgp_ctx* ctx, double* A, int ld, int n);
void dev_syrk_blocked(stgp_ctx* ctx, int n, long long k, double alpha, const double* A, int lda, double* C, int ldc,
                      int nb);
void dev_gemm_sym_blocked(stgp_ctx* ctx, int n, long long k, double alpha, const double* A, int lda, const double* B,
                          int ldb, double* C, int ldc, int nb);

}  // namespace stgp

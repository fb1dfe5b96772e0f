// FP64 GEMM emulated on the int8 tensor cores (ozaki.cu).
#pragma once

#include "common.cuh"

struct stgp_ctx;

namespace stgp {

struct OzakiState;
bool ozaki_enabled();
bool ozaki_for(int m);  // enabled and worth it at this inner size
int ozaki_slices();
// C[r * ldc + j] = sum_{c < k} A[r * lda + c] * B[j * ldb + c]  for r < n, j < m (FP64 in and out;
// m and ldc multiples of 4)
void ozaki_gemm_rows(stgp_ctx* ctx, long long n, int m, int k, const double* A, int lda, const double* B, int ldb,
                     double* C, int ldc);
// C = op(T) B for T lower triangular n x n (column-major, ldt) and B n x ncols (ldb): the rows form
// with the rows of op(T) as its per-row-scaled operand (n and ldc multiples of 4)
bool ozaki_trmm_enabled();
void ozaki_trmm_left(stgp_ctx* ctx, const double* T, int ldt, int n, const double* B, int ldb, long long ncols,
                     bool transpose, double* C, int ldc, bool skip = true);
// C[j * ldc + i] = sum_{r < n} A[j + r * lda] * B[i + r * ldb] / colD[r]  for i, j < m: A B^T of two
// m x n column-major matrices, each column scaled by colD[r]^{-1/2} when colD is given (the long
// reduction over n runs in exact int32 chunks)
void ozaki_gemm_cols(stgp_ctx* ctx, int m, long long n, const double* A, int lda, const double* B, int ldb, double* C,
                     int ldc, const double* colD = nullptr);
// K = (A D^{-1/2})(A D^{-1/2})^T keeping the digits of A D^{-1/2} in the context (tag: the owner's
// process-unique id, stgp_structure::uid);
// ozaki_gemm_kept then forms C[j ldc + i] = sum_r A[j, r] B[i, r] = (A D^{-1/2})(B D^{1/2})^T from
// them, slicing only B (false when the kept digits belong to another tag or shape).  symmetric: the
// product is known to be symmetric (FITC's W diag(phi) W^T): only the tiles reaching one triangle
// are computed and the other is mirrored.  colmul: an extra per-column factor of B (B(:, r) colmul_r),
// applied inside the slicer instead of in a separate pass over B.
void ozaki_syrk_keep(stgp_ctx* ctx, int m, long long n, const double* A, int lda, const double* D, double* C, int ldc,
                     uint64_t tag);
bool ozaki_gemm_kept(stgp_ctx* ctx, int m, long long n, const double* B, int ldb, const double* D, double* C, int ldc,
                     uint64_t tag, bool symmetric = false, const double* colmul = nullptr);
void ozaki_release(stgp_ctx* ctx);

// the hand-written tcgen05 kernel behind the products (ozaki_tc.cu)
struct OzakiTcState;
void ozaki_tc_release(OzakiTcState* s);
void ozaki_tc_rows(stgp_ctx* ctx, OzakiTcState*& st, int S, int kp, long long nx, int ny, const int8_t* xd, bool x_rev,
                   const double* sx, const int8_t* yd, bool y_rev, const double* sy, double* out, long long ldo,
                   int tri = 0);
void ozaki_tc_cols(stgp_ctx* ctx, OzakiTcState*& st, int S, int L, int nch, int m, const int8_t* xd, bool x_rev,
                   const double* sx, const int8_t* yd, bool y_rev, const double* sy, bool symmetric, double* C,
                   long long ldc);

}  // namespace stgp

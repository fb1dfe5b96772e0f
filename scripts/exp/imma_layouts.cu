// Which int8 IMMA operand layouts does cuBLASLt offer on this GPU, and how fast are they for the
// Ozaki long-reduction shape (912 x 912 output, K = 7 x 16384, batch 16)?  TN = K-major operands.
#include <cublasLt.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  cublasLtHandle_t lt; cublasLtCreate(&lt);
  const int m = 912, n = 912, k = 7 * 16384, batch = 16;
  int8_t *A, *B; int32_t* C; void* ws;
  const long long sa = (long long)m * k, sc = (long long)m * n;
  cudaMalloc(&A, sa * batch); cudaMalloc(&B, sa * batch); cudaMalloc(&C, sc * batch * 4); cudaMalloc(&ws, 64 << 20);
  cudaMemset(A, 1, sa * batch); cudaMemset(B, 1, sa * batch);
  for (int ta = 0; ta < 2; ++ta) for (int tb = 0; tb < 2; ++tb) {
    cublasLtMatmulDesc_t op; cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32I, CUDA_R_32I);
    cublasOperation_t a = ta ? CUBLAS_OP_T : CUBLAS_OP_N, b = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &a, sizeof a);
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &b, sizeof b);
    cublasLtMatrixLayout_t la, lb, lc;
    cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, ta ? k : m, ta ? m : k, ta ? k : m);
    cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, tb ? n : k, tb ? k : n, tb ? n : k);
    cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, m, n, m);
    for (auto l : {la, lb}) {
      cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof batch);
      cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof sa);
    }
    cublasLtMatrixLayoutSetAttribute(lc, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof batch);
    cublasLtMatrixLayoutSetAttribute(lc, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof sc);
    cublasLtMatmulPreference_t pref; cublasLtMatmulPreferenceCreate(&pref);
    size_t wss = 64 << 20; cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wss, sizeof wss);
    cublasLtMatmulHeuristicResult_t res[4]; int found = 0;
    cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 4, res, &found);
    const int one = 1, zero = 0;
    float best = 1e9;
    for (int i = 0; i < found; ++i) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cublasLtMatmul(lt, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[i].algo, ws, wss, 0);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) cublasLtMatmul(lt, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[i].algo, ws, wss, 0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      if (ms < best) best = ms;
    }
    printf("trans a=%c b=%c: algorithms %d, best %.3f ms = %.0f TOPS\n", ta ? 'T' : 'N', tb ? 'T' : 'N', found, best,
           2.0 * m * n * (double)k * batch / best / 1e9);
  }
  return 0;
}

// Experiment: CUTLASS RankK (DMMA, batched split-K) vs cuBLAS DGEMM for K = S S^T, S: 912 x 1.1M.
#include <cstdio>
#include <vector>
#include <cublas_v2.h>
#include "cutlass/cutlass.h"
#include "cutlass/gemm/device/rank_k.h"
#include "cutlass/epilogue/thread/linear_combination.h"

template <int TBM, int TBN, int WM, int WN, int STAGES>
using RankKT = cutlass::gemm::device::RankK<
    double, cutlass::layout::ColumnMajor, double, cutlass::layout::ColumnMajor, cutlass::FillMode::kLower, double,
    cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<TBM, TBN, 16>,
    cutlass::gemm::GemmShape<WM, WN, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<>, STAGES, 1, true, cutlass::arch::OpMultiplyAdd,
    cutlass::ComplexTransform::kNone, cutlass::BlasMode::kSymmetric>;

__global__ void fill(double* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = sin(0.001 * (double)(i % 100003)) * 0.1;
}

template <typename RK>
float run(const char* name, const double* A, int M, int ld, long long K, int P, double* part, cudaStream_t st) {
  typename RK::Arguments args(cutlass::gemm::GemmUniversalMode::kGemm, {M, M, (int)K}, P, {1.0, 0.0}, A, part,
                              part, 0, 0, 0, ld, ld, ld);
  RK op;
  cutlass::Status s = op.can_implement(args);
  if (s != cutlass::Status::kSuccess) { printf("%s: cannot implement\n", name); return -1; }
  size_t ws = RK::get_workspace_size(args);
  void* wsp = nullptr;
  if (ws) cudaMalloc(&wsp, ws);
  s = op.initialize(args, wsp, st);
  if (s != cutlass::Status::kSuccess) {
    printf("%s: init failed: %s (%s), ws=%zu\n", name, cutlassGetStatusString(s), cudaGetErrorString(cudaGetLastError()), ws);
    return -1;
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  s = op(st);
  if (s != cutlass::Status::kSuccess) printf("%s: run failed: %s (%s)\n", name, cutlassGetStatusString(s), cudaGetErrorString(cudaGetLastError()));
  cudaEventRecord(e0, st);
  for (int r = 0; r < 5; ++r) op(st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%s P=%d: %.2f ms  (%.1f TF/s on M^2 K)\n", name, P, ms / 5, (double)M * M * K / (ms / 5 * 1e-3) / 1e12);
  if (wsp) cudaFree(wsp);
  return ms / 5;
}

int main() {
  const int M = 912, ld = 912;
  const long long K = 1100000;
  double *A, *C, *part;
  cudaMalloc(&A, sizeof(double) * ld * K);
  cudaMalloc(&C, sizeof(double) * ld * ld);
  cudaMalloc(&part, sizeof(double) * ld * ld * 16);
  fill<<<4096, 256>>>(A, (long long)ld * K);
  cudaStream_t st; cudaStreamCreate(&st);
  cublasHandle_t h; cublasCreate(&h); cublasSetStream(h, st);
  const double one = 1.0, zero = 0.0;
  cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, M, M, (int)K, &one, A, ld, A, ld, &zero, C, ld);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int r = 0; r < 5; ++r) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, M, M, (int)K, &one, A, ld, A, ld, &zero, C, ld);
  cudaEventRecord(e1, st); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("cublas dgemm full: %.2f ms (%.1f TF/s on 2 M^2 K)\n", ms / 5, 2.0 * M * M * K / (ms / 5 * 1e-3) / 1e12);
  for (long long kk : {1024LL, 100000LL, 250000LL, 500000LL})
    run<RankKT<64, 64, 32, 32, 4>>("rankk 64x64 small-K", A, M, ld, kk, 4, part, st);
  for (int P : {4, 8, 16})
    run<RankKT<64, 64, 32, 32, 4>>("rankk 64x64 w32x32 s4", A, M, ld, K, P, part, st);
  for (int P : {4, 8})
    run<RankKT<128, 64, 64, 32, 3>>("rankk 128x64 w64x32 s3", A, M, ld, K, P, part, st);
  for (int P : {8, 16})
    run<RankKT<32, 32, 16, 16, 4>>("rankk 32x32 w16x16 s4", A, M, ld, K, P, part, st);
  // correctness of one partial sum vs cublas (lower triangle)
  std::vector<double> hc((size_t)ld * ld), hp((size_t)ld * ld * 4);
  run<RankKT<64, 64, 32, 32, 4>>("check", A, M, ld, K, 8, part, st);
  cudaMemcpy(hc.data(), C, sizeof(double) * ld * ld, cudaMemcpyDeviceToHost);
  cudaMemcpy(hp.data(), part, sizeof(double) * ld * ld, cudaMemcpyDeviceToHost);
  double maxrel = 0;
  for (int j = 0; j < M; ++j)
    for (int i = j; i < M; ++i) {
      double s = hp[(size_t)j * ld + i];
      const double c = hc[(size_t)j * ld + i];
      if (c != 0) maxrel = fmax(maxrel, fabs(s - c) / fabs(c));
    }
  printf("max rel diff vs cublas (lower): %.3e\n", maxrel);
  return 0;
}

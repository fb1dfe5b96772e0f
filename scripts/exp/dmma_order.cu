// Experiment: is mma.sync m8n8k4 f64 bit-identical to a sequential fma chain over k?
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <random>
#include <vector>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// A: 8 x K row-major, B: K x 8 (col-major = B^T row-major 8 x K). C = A B, K multiple of 4.
__global__ void k_mma(const double* A, const double* B, int K, double* C) {
  const int lane = threadIdx.x, grp = lane >> 2, tig = lane & 3;
  double d0 = 0, d1 = 0;
  for (int kb = 0; kb < K; kb += 4) dmma(d0, d1, A[grp * K + kb + tig], B[grp * K + kb + tig]);
  C[grp * 8 + 2 * tig] = d0;
  C[grp * 8 + 2 * tig + 1] = d1;
}
__global__ void k_seq(const double* A, const double* B, int K, double* C, int variant) {
  const int r = threadIdx.x / 8, c = threadIdx.x % 8;
  double s = 0;
  if (variant == 0) {
    for (int k = 0; k < K; ++k) s = __fma_rn(A[r * K + k], B[c * K + k], s);
  } else {  // per-4 block: products summed then added? (pairwise within k-step)
    for (int kb = 0; kb < K; kb += 4) {
      double p = __dmul_rn(A[r * K + kb], B[c * K + kb]);
      for (int t = 1; t < 4; ++t) p = __fma_rn(A[r * K + kb + t], B[c * K + kb + t], p);
      s = __dadd_rn(s, p);
    }
  }
  C[r * 8 + c] = s;
}
int main() {
  const int K = 912, trials = 2000;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::vector<double> hA(8 * K), hB(8 * K), c1(64), c2(64), c3(64);
  double *A, *B, *C;
  cudaMalloc(&A, 8 * K * 8); cudaMalloc(&B, 8 * K * 8); cudaMalloc(&C, 64 * 8);
  long long eq0 = 0, eq1 = 0, tot = 0;
  double maxrel = 0;
  for (int t = 0; t < trials; ++t) {
    for (auto& v : hA) v = nd(g) * std::exp(nd(g) * 3);
    for (auto& v : hB) v = nd(g) * std::exp(nd(g) * 3);
    cudaMemcpy(A, hA.data(), 8 * K * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB.data(), 8 * K * 8, cudaMemcpyHostToDevice);
    k_mma<<<1, 32>>>(A, B, K, C); cudaMemcpy(c1.data(), C, 64 * 8, cudaMemcpyDeviceToHost);
    k_seq<<<1, 64>>>(A, B, K, C, 0); cudaMemcpy(c2.data(), C, 64 * 8, cudaMemcpyDeviceToHost);
    k_seq<<<1, 64>>>(A, B, K, C, 1); cudaMemcpy(c3.data(), C, 64 * 8, cudaMemcpyDeviceToHost);
    for (int e = 0; e < 64; ++e) {
      eq0 += c1[e] == c2[e];
      eq1 += c1[e] == c3[e];
      ++tot;
      if (c2[e] != 0) maxrel = std::fmax(maxrel, std::fabs(c1[e] - c2[e]) / std::fabs(c2[e]));
    }
  }
  printf("dmma == sequential fma chain: %lld / %lld\n", eq0, tot);
  printf("dmma == per-kstep (mul + fma x3) then add: %lld / %lld\n", eq1, tot);
  printf("max rel diff vs chain %.3e\n", maxrel);
  return 0;
}

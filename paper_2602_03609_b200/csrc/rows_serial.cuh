// Generic per-row path for conditioning sets larger than a warp (k > 31), e.g.
// the full-conditioning exactness tests (test_approximations.cpp:78-142); all four modes, including
// the VIF gradient's per-row pass.
// One thread per row, the k x k block in a per-thread global scratch slab.
// Same semantics as rows.cuh; throughput is irrelevant at these sizes.
#pragma once
// The per-mode early exits (`if (MODE == kModeBuild) continue;`) make the rest of the loop body dead
// in that instantiation by design; silence the resulting "loop is not reachable" note.
#pragma nv_diag_suppress 128

#include "rows.cuh"

namespace stgp {

template <int MODE, bool HAS_W>
__global__ void __launch_bounds__(64) vecchia_rows_serial_kernel(RowArgs a, double* scratch) {
  const int K = a.m_v;
  const size_t slab = static_cast<size_t>(K) * K + 8 * static_cast<size_t>(K) + 16;
  double tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int tidg = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  double* C = scratch + static_cast<size_t>(tidg) * slab;
  double* c = C + static_cast<size_t>(K) * K;
  double* A = c + K;
  double* wv = A + K;
  double* rn = wv + K;
  double* tcl = rn + K;   // a~ over the closure (K + 1)
  double* wcl = tcl + K + 1;
  int* N = reinterpret_cast<int*>(wcl + K + 1);  // K ints (fits in 2K doubles)
  auto cov = [&](int p, int q) {
    double pe, pb;
    a.lt.get2(a.tid[p], a.tid[q], pe, pb);
    TF f;
    f.pow_mE = pe;
    f.pow_mbh = pb;
    double v = gneiting_eval<true>(a.k, spatial_dist(a.x[p], a.y[p], a.x[q], a.y[q]), f);
    if (HAS_W) {
      double s = 0.0;
      for (int j = 0; j < a.ldw; ++j) s = fma(a.W[static_cast<size_t>(p) * a.ldw + j], a.W[static_cast<size_t>(q) * a.ldw + j], s);
      v = __dsub_rn(v, s);
    }
    if (p == q) v = __dadd_rn(v, a.nugget);
    return v;
  };
  for (int i = a.row_begin + tidg; i < a.row_end; i += nt) {
    int k = 0;
    while (k < K && a.nbr[static_cast<size_t>(i) * K + k] >= 0) {
      N[k] = a.nbr[static_cast<size_t>(i) * K + k];
      ++k;
    }
    for (int p = 0; p < k; ++p) {
      c[p] = cov(i, N[p]);
      for (int q = 0; q <= p; ++q) {
        const double v = cov(N[p], N[q]);
        C[p * K + q] = v;
        C[q * K + p] = v;
      }
    }
    const double dii = cov(i, i);
    // Cholesky (lower, in place in the lower triangle; upper keeps C) with jitter ladder
    bool ok = false;
    double* L = C;  // reuse: factor written to lower triangle, diagonal saved in A[] temporarily
    for (int attempt = 0; attempt < 3 && !ok; ++attempt) {
      // restore lower triangle from the (symmetric) upper triangle and diagonal copy
      for (int p = 0; p < k; ++p) {
        for (int q = 0; q < p; ++q) L[p * K + q] = C[q * K + p];
        if (attempt == 0) wv[p] = C[p * K + p];  // keep the original diagonal
        double d = wv[p];
        if (attempt >= 1) d = __dadd_rn(d, 1e-10 * a.s1);
        if (attempt == 2) d = __dadd_rn(d, 9.0 * (1e-10 * a.s1));
        L[p * K + p] = d;
      }
      bool good = true;
      for (int j = 0; j < k && good; ++j) {
        double s = L[j * K + j];
        for (int m = 0; m < j; ++m) s = fma(-L[j * K + m], L[j * K + m], s);
        if (!(s > 0.0) && s <= 0.0) {
          good = false;
          break;
        }
        const double d = sqrt(s);
        L[j * K + j] = d;
        for (int r = j + 1; r < k; ++r) {
          double t = L[r * K + j];
          for (int m = 0; m < j; ++m) t = fma(-L[r * K + m], L[j * K + m], t);
          L[r * K + j] = t / d;
        }
      }
      ok = good;
    }
    if (!ok) {
      atomicMin(a.fail_row, i);
      continue;
    }
    auto solve = [&](const double* b, double* x) {
      for (int r = 0; r < k; ++r) {
        double s = b[r];
        for (int m = 0; m < r; ++m) s = fma(-L[r * K + m], x[m], s);
        x[r] = s / L[r * K + r];
      }
      for (int r = k - 1; r >= 0; --r) {
        double s = x[r];
        for (int m = r + 1; m < k; ++m) s = fma(-L[m * K + r], x[m], s);
        x[r] = s / L[r * K + r];
      }
    };
    solve(c, A);
    double ac = 0.0;
    for (int p = 0; p < k; ++p) ac += A[p] * c[p];
    const double D = dii - ac;
    if (!(D > 0.0)) {
      atomicMin(a.fail_row, i);
      continue;
    }
    if (a.A_out)
      for (int p = 0; p < K; ++p) a.A_out[static_cast<size_t>(i) * K + p] = p < k ? A[p] : 0.0;
    if (a.D_out) a.D_out[i] = D;
    if (MODE == kModeBuild) continue;
    double u = a.r[i];
    for (int p = 0; p < k; ++p) u -= A[p] * a.r[N[p]];
    tot[0] += log(D) + u * u / D;
    if (MODE != kModeGrad && MODE != kModeVifGrad) continue;
    double cd, cu;
    if (MODE == kModeVifGrad) {
      // Rv = C^{-1} vrow_N with vrow_p = (W_{N_p} . X_i + Bz_i z_{N_p}) / D_i, and
      // Phi_i = c0 a~a~' - sym(a~ Rv')   (approximations.cpp:616-661; rows.cuh kModeVifGrad)
      const double Dst = a.D_in[i], uz = a.Bz[i];
      const double* xi = a.X + static_cast<size_t>(i) * a.ldw;
      for (int p = 0; p < k; ++p) {
        const double* wp = a.W + static_cast<size_t>(N[p]) * a.ldw;
        double ga = 0.0;
        for (int j = 0; j < a.ldw; ++j) ga = fma(wp[j], xi[j], ga);
        rn[p] = (ga + uz * a.z[N[p]]) / Dst;
      }
      solve(rn, wv);
      const double* vi = a.Vp + static_cast<size_t>(i) * a.ldw;
      double aGa = 0.0;
      for (int j = 0; j < a.ldw; ++j) aGa = fma(vi[j], xi[j], aGa);
      cd = 0.5 * (1.0 / Dst - (aGa + uz * uz) / (Dst * Dst));
      cu = 1.0;
      a.c0_out[i] = cd;
      for (int p = 0; p < K; ++p) a.Rv_out[static_cast<size_t>(i) * K + p] = p < k ? wv[p] : 0.0;
    } else {
      for (int p = 0; p < k; ++p) rn[p] = a.r[N[p]];
      solve(rn, wv);
      cd = 0.5 * (1.0 / D - u * u / (D * D));
      cu = u / D;
    }
    double aa = 0.0, aw = 0.0;
    for (int p = 0; p < k; ++p) {
      aa += A[p] * A[p];
      aw += A[p] * wv[p];
      tcl[p] = -A[p];
      wcl[p] = wv[p];
    }
    tcl[k] = 1.0;
    wcl[k] = 0.0;
    double g[6] = {0, 0, 0, 0, 0, 0};
    for (int p = 1; p <= k; ++p) {
      const int pp = p < k ? N[p] : i;
      for (int q = 0; q < p; ++q) {
        const int qq = N[q];
        const TF f = a.lt.get(a.tid[pp], a.tid[qq]);
        double kg[6];
        gneiting_grad(a.k, spatial_dist(a.x[pp], a.y[pp], a.x[qq], a.y[qq]), f, kg);
        const double wt = cd * (2.0 * tcl[p] * tcl[q]) - cu * (wcl[p] * tcl[q] + wcl[q] * tcl[p]);
        for (int s = 0; s < 6; ++s) g[s] = fma(wt, kg[s], g[s]);
      }
    }
    const double wd = cd * (1.0 + aa) - cu * (-aw);
    tot[1] += wd;
    for (int s = 0; s < 6; ++s) tot[2 + s] += g[s] + wd * a.g00[s];
  }
  // per-thread partials -> per-block in thread order (deterministic)
  __shared__ double red[64][8];
  for (int q = 0; q < 8; ++q) red[threadIdx.x][q] = tot[q];
  __syncthreads();
  if (threadIdx.x < 8) {
    double s = 0.0;
    for (int t = 0; t < static_cast<int>(blockDim.x); ++t) s += red[t][threadIdx.x];
    a.part[static_cast<size_t>(blockIdx.x) * 8 + threadIdx.x] = s;
  }
}

}  // namespace stgp

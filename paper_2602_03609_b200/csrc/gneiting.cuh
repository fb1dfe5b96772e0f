// Device Gneiting space-time kernel (reference covariance.cpp:62-181).
//
// Bit-exactness contract: every operation below is an explicit IEEE
// round-to-nearest intrinsic in the reference's evaluation order, so a device
// covariance equals the host `GneitingKernel::eval` bit-for-bit given the same
// temporal factors.  Temporal factors (pow/log of the time lag) are computed on
// the host with glibc and tabulated per time-id pair; the only transcendental
// left on the device is exp, ported from glibc 2.39's FMA variant
// (sysdeps/ieee754/dbl-64/e_exp.c, compiled by glibc with -mfma -mavx2).
#pragma once

#include <cstdint>

#include "common.cuh"
#include "glibc_exp_table.h"

namespace stgp {

// global table (per translation unit): divergent indexed loads, constant memory would serialise them
static __device__ uint64_t kExpTab[256] = STGP_EXP_TABLE_INIT;

// glibc exp, specialcase(): k > 0 keeps the contracted form; k < 0 shares the
// product scale*tmp (GCC CSE), so nothing there is contracted.
static __device__ __noinline__ double glibc_exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ULL) == 0) {
    sbits -= 1009ULL << 52;
    const double scale = __longlong_as_double(static_cast<long long>(sbits));
    return __dmul_rn(0x1p1009, __fma_rn(scale, tmp, scale));
  }
  sbits += 1022ULL << 52;
  const double scale = __longlong_as_double(static_cast<long long>(sbits));
  const double st = __dmul_rn(scale, tmp);
  double y = __dadd_rn(scale, st);
  if (y < 1.0) {
    double lo = __dadd_rn(__dsub_rn(scale, y), st);
    const double hi = __dadd_rn(1.0, y);
    lo = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
    y = __dsub_rn(__dadd_rn(hi, lo), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return __dmul_rn(0x1p-1022, y);
}

__device__ __forceinline__ double glibc_exp(double x) {
  const uint64_t ux = static_cast<uint64_t>(__double_as_longlong(x));
  uint32_t abstop = static_cast<uint32_t>(ux >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
    if (abstop - 0x3c9u >= 0x80000000u) return __dadd_rn(1.0, x);  // |x| < 2^-54
    if (abstop >= 0x409u) {
      if (ux == 0xfff0000000000000ULL) return 0.0;
      if (abstop >= 0x7ffu) return __dadd_rn(1.0, x);
      return (ux >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
    }
    abstop = 0;  // large |x|: special case below
  }
  double kd = __fma_rn(STGP_EXP_invln2N, x, STGP_EXP_shift);
  const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
  kd = __dsub_rn(kd, STGP_EXP_shift);
  const double r = __fma_rn(kd, STGP_EXP_negln2loN, __fma_rn(kd, STGP_EXP_negln2hiN, x));
  const uint32_t idx = 2u * static_cast<uint32_t>(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = __longlong_as_double(static_cast<long long>(__ldg(&kExpTab[idx])));
  const uint64_t sbits = __ldg(&kExpTab[idx + 1]) + top;
  const double r2 = __dmul_rn(r, r);
  const double tmp =
      __fma_rn(__dmul_rn(r2, r2), __fma_rn(r, STGP_EXP_C5, STGP_EXP_C4),
               __fma_rn(r2, __fma_rn(r, STGP_EXP_C3, STGP_EXP_C2), __dadd_rn(tail, r)));
  if (abstop == 0) return glibc_exp_special(tmp, sbits, ki);
  const double scale = __longlong_as_double(static_cast<long long>(sbits));
  return __fma_rn(scale, tmp, scale);
}

// spatial distance, types.hpp:53-56
__device__ __forceinline__ double spatial_dist(double xa, double ya, double xb, double yb) {
  const double dx = __dsub_rn(xa, xb), dy = __dsub_rn(ya, yb);
  return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
}

// Matern correlation for nu in {0.5, 1.5, 2.5} (covariance.cpp:66-71), given e = exp(-x)
__device__ __forceinline__ double matern_from_exp(double x, double e, int nu_code) {
  if (x == 0.0) return 1.0;
  if (nu_code == 0) return e;
  if (nu_code == 1) return __dmul_rn(__dadd_rn(1.0, x), e);
  return __dmul_rn(__dadd_rn(__dadd_rn(1.0, x), __ddiv_rn(__dmul_rn(x, x), 3.0)), e);
}
// derivative (covariance.cpp:79-87)
__device__ __forceinline__ double matern_deriv_from_exp(double x, double e, int nu_code) {
  if (nu_code == 0) return -e;
  if (nu_code == 1) return __dmul_rn(-x, e);
  return __dmul_rn(-__ddiv_rn(__dmul_rn(x, __dadd_rn(1.0, x)), 3.0), e);
}

constexpr int kNuGeneral = 3;  // nu outside {0.5, 1.5, 2.5}: Bessel-K form, value only

// nu-only constants of the general Matern (host-computed with glibc, MaternNu::make in engine.cu):
// K_nu is evaluated at mu = nu - nl (|mu| <= 1/2) and raised to nu by the upward recurrence.
struct MaternNu {
  double nu, mu, coef;           // coef = 2^(1-nu) / Gamma(nu)   (covariance.cpp:73-74)
  double gam1, gam2, gampl, gammi, fact;  // Temme's Gamma combinations at mu; fact = pi mu / sin(pi mu)
  int nl;
};

struct DevKernel {
  double s1, c, a, beta, E;  // sigma1_2, spatial decay, temporal scale, beta, delta+beta
  int nu_code;               // 0: 0.5, 1: 1.5, 2: 2.5, kNuGeneral: other (eval only)
  MaternNu g;                // used when nu_code == kNuGeneral
};

inline int nu_code_of(double nu) {
  if (nu == 0.5) return 0;
  if (nu == 1.5) return 1;
  if (nu == 2.5) return 2;
  return kNuGeneral;
}

// K_mu(x), K_{mu+1}(x) for |mu| <= 1/2, x > 0: Temme's series below x = 2, Steed's continued
// fraction CF2 (Temme's normalisation) above -- the method of the libstdc++ std::cyl_bessel_k the
// reference calls (covariance.cpp:74), evaluated here with CUDA's log/exp/sinh/cosh (a few ulp,
// so general-nu covariances match the reference to ~1e-15 relative, not bit for bit).
__device__ __forceinline__ double bessel_k_nu(const MaternNu& g, double x) {
  constexpr double kEps = 2.220446049250313e-16;
  constexpr int kMaxIter = 15000;
  const double mu = g.mu, xi = 1.0 / x, xi2 = 2.0 * xi;
  double kmu, kmu1;
  if (x < 2.0) {
    const double x2 = 0.5 * x;
    double d = -log(x2);
    double e = mu * d;
    const double fact2 = fabs(e) < kEps ? 1.0 : sinh(e) / e;
    double ff = g.fact * (g.gam1 * cosh(e) + g.gam2 * fact2 * d);
    double sum = ff;
    e = exp(e);
    double p = 0.5 * e / g.gampl, q = 0.5 / (e * g.gammi), c = 1.0;
    d = x2 * x2;
    double sum1 = p;
    for (int i = 1; i <= kMaxIter; ++i) {
      const double di = static_cast<double>(i);
      ff = (di * ff + p + q) / (di * di - mu * mu);
      c *= d / di;
      p /= di - mu;
      q /= di + mu;
      const double del = c * ff;
      sum += del;
      sum1 += c * (p - di * ff);
      if (fabs(del) < kEps * fabs(sum)) break;
    }
    kmu = sum;
    kmu1 = sum1 * xi2;
  } else {
    double b = 2.0 * (1.0 + x), d = 1.0 / b, h = d, delh = d, q1 = 0.0, q2 = 1.0;
    const double a1 = 0.25 - mu * mu;
    double q = a1, c = a1, a = -a1, s = 1.0 + q * delh;
    for (int i = 2; i <= kMaxIter; ++i) {
      a -= 2.0 * (i - 1);
      c = -a * c / i;
      const double qnew = (q1 - b * q2) / a;
      q1 = q2;
      q2 = qnew;
      q += c * qnew;
      b += 2.0;
      d = 1.0 / (b + a * d);
      delh = (b * d - 1.0) * delh;
      h += delh;
      const double dels = q * delh;
      s += dels;
      if (fabs(dels / s) < kEps) break;
    }
    h = a1 * h;
    kmu = sqrt(3.141592653589793 / (2.0 * x)) * exp(-x) / s;
    kmu1 = kmu * (mu + x + 0.5 - h) * xi;
  }
  for (int i = 1; i <= g.nl; ++i) {  // K_{mu+i+1} = 2 (mu+i)/x K_{mu+i} + K_{mu+i-1}
    const double kn = (mu + i) * xi2 * kmu1 + kmu;
    kmu = kmu1;
    kmu1 = kn;
  }
  return kmu;
}

// matern_corr for general nu (covariance.cpp:72-76): 2^(1-nu)/Gamma(nu) x^nu K_nu(x), 0 where
// K_nu underflows
// (out of line: the closed-form kernels keep their registers; only this branch pays the call)
static __device__ __noinline__ double matern_general(const MaternNu& g, double x) {
  if (x == 0.0) return 1.0;
  const double v = g.coef * pow(x, g.nu) * bessel_k_nu(g, x);
  return isfinite(v) ? v : 0.0;
}

// GneitingKernel::eval (covariance.cpp:138-149).  GEN = false compiles the closed forms only (the
// hot kernels' default: the out-of-line general branch costs them registers); kernels that can see a
// general nu are instantiated with GEN = true by their launchers.
template <bool GEN = false>
__device__ __forceinline__ double gneiting_eval(const DevKernel& k, double h, const TF& f) {
  const double x = __dmul_rn(__dmul_rn(k.c, h), f.pow_mbh);
  if (GEN && k.nu_code == kNuGeneral) return __dmul_rn(__dmul_rn(k.s1, f.pow_mE), matern_general(k.g, x));
  const double e = (x == 0.0) ? 1.0 : glibc_exp(-x);
  return __dmul_rn(__dmul_rn(k.s1, f.pow_mE), matern_from_exp(x, e, k.nu_code));
}

// GneitingKernel::grad (covariance.cpp:151-181); g order (sigma1_2, a, c, alpha, beta, delta).
// Also returns the covariance value.
__device__ __forceinline__ double gneiting_grad(const DevKernel& k, double h, const TF& f, double g[6]) {
  const double x = __dmul_rn(__dmul_rn(k.c, h), f.pow_mbh);
  const double e = glibc_exp(-x);
  const double M = matern_from_exp(x, e, k.nu_code);
  const double Mp = matern_deriv_from_exp(x, e, k.nu_code);
  const double base = __dmul_rn(k.s1, f.pow_mE);
  g[0] = __dmul_rn(f.pow_mE, M);
  const double dC_dT = __dmul_rn(__dmul_rn(base, f.inv_T),
                                 __dsub_rn(__dmul_rn(-k.E, M), __dmul_rn(__dmul_rn(__dmul_rn(0.5, k.beta), x), Mp)));
  g[1] = __dmul_rn(dC_dT, f.u2a);
  g[3] = __dmul_rn(__dmul_rn(__dmul_rn(dC_dT, 2.0), k.a), f.u2a_logu);
  g[2] = __ddiv_rn(__dmul_rn(__dmul_rn(base, Mp), x), k.c);
  g[4] = __dmul_rn(__dmul_rn(-f.log_T, base), __dadd_rn(M, __dmul_rn(__dmul_rn(0.5, x), Mp)));
  g[5] = __dmul_rn(__dmul_rn(-f.log_T, base), M);
  return __dmul_rn(base, M);
}

// Gradient with the divisions replaced by precomputed reciprocals (inv_c = 1/c);
// used where only the 1e-8 tolerance applies (likelihood gradients).
__device__ __forceinline__ void gneiting_grad_fast(const DevKernel& k, double inv_c, double h, const TF& f,
                                                   double g[6]) {
  const double x = k.c * h * f.pow_mbh;
  const double e = glibc_exp(-x);
  double M, Mp;
  if (k.nu_code == 0) {
    M = e;
    Mp = -e;
  } else if (k.nu_code == 1) {
    M = (1.0 + x) * e;
    Mp = -x * e;
  } else {
    M = (1.0 + x + x * x * (1.0 / 3.0)) * e;
    Mp = -(x * (1.0 + x) * (1.0 / 3.0)) * e;
  }
  if (x == 0.0) M = 1.0;
  const double base = k.s1 * f.pow_mE;
  g[0] = f.pow_mE * M;
  const double dC_dT = base * f.inv_T * (-k.E * M - 0.5 * k.beta * x * Mp);
  g[1] = dC_dT * f.u2a;
  g[3] = dC_dT * 2.0 * k.a * f.u2a_logu;
  g[2] = base * Mp * x * inv_c;
  g[4] = -f.log_T * base * (M + 0.5 * x * Mp);
  g[5] = -f.log_T * base * M;
}

// ---- branch-free pieces for the likelihood-gradient pair loops (1e-8 tolerance) ----
// No special-case paths, so the scheduler can interleave several pairs' dependency chains.

// sqrt(s), s >= 0, within ~1 ulp: approximate rsqrt, two Newton steps, one residual correction;
// s below DBL_MIN maps to 0 (a distance under 1e-154: the kernel is at its x = 0 value anyway).
__device__ __forceinline__ double sqrt_nr(double s) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  const double hs = 0.5 * s;
  y = y * fma(-hs, y * y, 1.5);
  y = y * fma(-hs, y * y, 1.5);
  double h = s * y;
  h = fma(fma(-h, h, s), 0.5 * y, h);
  return s >= 2.2250738585072014e-308 ? h : 0.0;
}

// exp(t) for t <= 0: glibc's table method without its special cases; t is clamped at -708 (results
// below 3e-308 only ever scale gradient terms that are already negligible), within ~1 ulp otherwise.
__device__ __forceinline__ double exp_nonpos(double t) {
  t = fmax(t, -708.0);
  double kd = fma(STGP_EXP_invln2N, t, STGP_EXP_shift);
  const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
  kd -= STGP_EXP_shift;
  const double r = fma(kd, STGP_EXP_negln2loN, fma(kd, STGP_EXP_negln2hiN, t));
  const uint32_t idx = 2u * static_cast<uint32_t>(ki & 127u);
  const double tail = __longlong_as_double(static_cast<long long>(__ldg(&kExpTab[idx])));
  const uint64_t sbits = __ldg(&kExpTab[idx + 1]) + (ki << 45);
  const double r2 = r * r;
  const double tmp = fma(r2 * r2, fma(r, STGP_EXP_C5, STGP_EXP_C4), fma(r2, fma(r, STGP_EXP_C3, STGP_EXP_C2), tail + r));
  const double scale = __longlong_as_double(static_cast<long long>(sbits));
  return fma(scale, tmp, scale);
}

// Matern M = (1 + m1 x + m2 x^2) e and M' = -(p0 + p1 x + p2 x^2) e for the closed forms
struct MaternPoly {
  double m1, m2, p0, p1, p2;
};
__host__ __device__ inline MaternPoly matern_poly(int nu_code) {
  if (nu_code == 0) return MaternPoly{0.0, 0.0, 1.0, 0.0, 0.0};
  if (nu_code == 1) return MaternPoly{1.0, 0.0, 0.0, 1.0, 0.0};
  return MaternPoly{1.0, 1.0 / 3.0, 0.0, 1.0 / 3.0, 1.0 / 3.0};
}

// gneiting_grad_fast from the squared distance, branch free (same formulas, ~ulp-level differences)
__device__ __forceinline__ void gneiting_grad_bf(const DevKernel& k, const MaternPoly& mp, double inv_c, double s,
                                                 const TF& f, double g[6]) {
  const double x = k.c * sqrt_nr(s) * f.pow_mbh;
  const double e = exp_nonpos(-x);
  const double M = fma(fma(mp.m2, x, mp.m1), x, 1.0) * e;
  const double Mp = -fma(fma(mp.p2, x, mp.p1), x, mp.p0) * e;
  const double base = k.s1 * f.pow_mE;
  g[0] = f.pow_mE * M;
  const double dC_dT = base * f.inv_T * (-k.E * M - 0.5 * k.beta * x * Mp);
  g[1] = dC_dT * f.u2a;
  g[3] = dC_dT * 2.0 * k.a * f.u2a_logu;
  g[2] = base * Mp * x * inv_c;
  g[4] = -f.log_T * base * (M + 0.5 * x * Mp);
  g[5] = -f.log_T * base * M;
}

// Covariance from the squared distance with the branch-free pieces (closed-form Matern only): within a
// few ulp of gneiting_eval; for the likelihood-gradient passes, where only the 1e-8 tolerance applies.
__device__ __forceinline__ double gneiting_eval_bf(const DevKernel& k, const MaternPoly& mp, double s, const TF& f) {
  const double x = k.c * sqrt_nr(s) * f.pow_mbh;
  const double e = exp_nonpos(-x);
  return k.s1 * f.pow_mE * (fma(fma(mp.m2, x, mp.m1), x, 1.0) * e);
}

// Temporal-factor table indexed by time-id pairs (host-computed with glibc).
struct TFTable {
  const TF* tab;  // nT * nT
  int nT;
  __device__ __forceinline__ TF get(int ta, int tb) const {
    const TF* p = tab + static_cast<size_t>(ta) * nT + tb;
    TF f;
    f.pow_mE = __ldg(&p->pow_mE);
    f.pow_mbh = __ldg(&p->pow_mbh);
    f.inv_T = __ldg(&p->inv_T);
    f.log_T = __ldg(&p->log_T);
    f.u2a = __ldg(&p->u2a);
    f.u2a_logu = __ldg(&p->u2a_logu);
    return f;
  }
  __device__ __forceinline__ void get2(int ta, int tb, double& pow_mE, double& pow_mbh) const {
    const TF* p = tab + static_cast<size_t>(ta) * nT + tb;
    pow_mE = __ldg(&p->pow_mE);
    pow_mbh = __ldg(&p->pow_mbh);
  }
};

// Covariance between two points given their time ids.
__device__ __forceinline__ double cov_pts(const DevKernel& k, const TFTable& T, double xa, double ya,
                                          int ta, double xb, double yb, int tb) {
  TF f;
  T.get2(ta, tb, f.pow_mE, f.pow_mbh);
  return gneiting_eval(k, spatial_dist(xa, ya, xb, yb), f);
}

}  // namespace stgp

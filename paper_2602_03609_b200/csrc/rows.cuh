// Per-observation Vecchia/VIF row kernels (K1, K1g, K3 of SURVEY.md §2.4).
//
// One warp per row i.  Closure slots: 0..k-1 hold N(i) (ascending), k..KS-1 are
// identity padding, slot KS holds i itself (KS >= m_v is a compile-time size,
// KS <= 31).  Lane r owns row r of the KS x KS conditioning block in registers.
//   phase A  pairwise Gneiting covariances of the closure, lane-strided over a
//            shared pair table, into shared memory; VIF: minus the closure Gram
//            W_cl^T W_cl computed with FP64 DMMA (mma.sync m8n8k4 f64) straight
//            from the column-major W in HBM/L2;
//   phase B  right-looking Cholesky in registers: pivot broadcast by shuffle,
//            1/sqrt once per column, L column broadcast through shared memory;
//            the reference's jitter ladder (approximations.cpp:91-103);
//   phase C  A_i = C^{-1} c, D_i = d_ii - A.c (approximations.cpp:104-110),
//            u_i = (B r)_i, NLL term log D_i + u_i^2 / D_i (approximations.cpp:340-346);
//   phase D  (gradient) kernel gradients over closure pairs weighted by
//            c_d a~a~' - c_u sym(w~ a~') (approximations.cpp:419-483).
// Per-row results are reduced per block in a fixed order (deterministic).
#pragma once

#include "common.cuh"
#include "gneiting.cuh"

namespace stgp {

constexpr int kRowWarps = 4;
constexpr int kKmax = 32;  // closure slots per warp (k <= 31 neighbours)
constexpr unsigned kFull = 0xffffffffu;

// Temporal factors of a time-id pair.  Table mode (nT <= 4096 distinct times): lagid[ta nT + tb] indexes
// the host-tabulated factors of the distinct lags.  Live mode (more distinct times): u = |T[ta] - T[tb]|,
// the structure's integer-lag table when it applies (covariance.cpp:127-146 snap rule, host glibc:
// bit-identical to the table mode), otherwise the factors evaluated on the device (covariance.cpp:94-113
// with CUDA's pow / log: within a few ulp of glibc).
struct LagTable {
  const int32_t* lagid;  // nT * nT -> index into tf (table mode), or null (live mode)
  const TF* tf;
  int nT;
  const double* Tv;   // live mode: the time value of each id
  const TF* itab;     // live mode: integer-lag table (null when the policy has none)
  int itab_n;
  double la, two_alpha, E, half_beta;  // live mode: a, 2 alpha, delta + beta, beta / 2
  // out of line: the table-mode fast path of get / get2 stays small (register pressure of the hot kernels)
  __device__ __noinline__ TF live(double u) const {
    TF f;
    if (u == 0.0) {
      f.pow_mE = 1.0;
      f.pow_mbh = 1.0;
      f.inv_T = 1.0;
      f.log_T = 0.0;
      f.u2a = 0.0;
      f.u2a_logu = 0.0;
      return f;
    }
    const double r = nearbyint(u);
    if (itab && fabs(u - r) < 1e-9 && r < static_cast<double>(itab_n)) {
      const TF* p = itab + static_cast<int>(r);
      f.pow_mE = __ldg(&p->pow_mE);
      f.pow_mbh = __ldg(&p->pow_mbh);
      f.inv_T = __ldg(&p->inv_T);
      f.log_T = __ldg(&p->log_T);
      f.u2a = __ldg(&p->u2a);
      f.u2a_logu = __ldg(&p->u2a_logu);
      return f;
    }
    f.u2a = pow(u, two_alpha);
    f.u2a_logu = f.u2a * log(u);
    const double T = la * f.u2a + 1.0;
    f.inv_T = 1.0 / T;
    f.log_T = log(T);
    f.pow_mE = pow(T, -E);
    f.pow_mbh = pow(T, -half_beta);
    return f;
  }
  __device__ __forceinline__ double lag(int ta, int tb) const { return fabs(__ldg(&Tv[ta]) - __ldg(&Tv[tb])); }
  __device__ __forceinline__ const TF* at(int ta, int tb) const {
    return tf + __ldg(&lagid[static_cast<size_t>(ta) * nT + tb]);
  }
  __device__ __forceinline__ void get2(int ta, int tb, double& pow_mE, double& pow_mbh) const {
    if (!lagid) {
      const TF f = live(lag(ta, tb));
      pow_mE = f.pow_mE;
      pow_mbh = f.pow_mbh;
      return;
    }
    const TF* p = at(ta, tb);
    pow_mE = __ldg(&p->pow_mE);
    pow_mbh = __ldg(&p->pow_mbh);
  }
  __device__ __forceinline__ TF get(int ta, int tb) const {
    if (!lagid) return live(lag(ta, tb));
    const TF* p = at(ta, tb);
    TF f;
    f.pow_mE = __ldg(&p->pow_mE);
    f.pow_mbh = __ldg(&p->pow_mbh);
    f.inv_T = __ldg(&p->inv_T);
    f.log_T = __ldg(&p->log_T);
    f.u2a = __ldg(&p->u2a);
    f.u2a_logu = __ldg(&p->u2a_logu);
    return f;
  }
};

struct RowArgs {
  int n, m_v;
  int row_begin, row_end;  // rows processed [row_begin, row_end)
  const int32_t* order;    // optional locality schedule: the k-th row processed is order[k]
  unsigned long long* next;  // optional: rows claimed in order from this (zeroed) counter
  double* row_part;          // optional: per-row contributions [(i - row_begin) * 8 + q] instead of tot
  const int32_t* nbr;      // n * m_v, ascending, -1 padded
  const double *x, *y;
  const int32_t* tid;
  DevKernel k;
  LagTable lt;
  double s1;      // sigma1_2
  double nugget;  // added to block diagonals (policy)
  // VIF: whitened cross covariance, column-major ldw x n (rows >= M are 0)
  const double* W;
  int ldw;
  const double* zcol;  // ldw zeros: the fragment source of empty closure slots (no load predicates)
  const double* r;  // residual y - X beta (NLL / gradient modes)
  double* A_out;    // n * m_v (optional)
  double* D_out;    // n (optional)
  double* u_out;    // n (optional): u_i = (B r)_i
  double* part;     // per-block partial sums [gridDim.x][8]
  int* fail_row;    // min failing row index (init INT_MAX)
  double g00[6];    // kernel gradient at (h, u) = (0, 0)
  double inv_c;     // 1 / c
  // VIF gradient mode (approximations.cpp:616-661): X = K^{-1} V' (ldw x n),
  // Vp = V' = W B^T, z = r - t, Bz = B z, D from the build; outputs c0, Rv.
  const double* X;
  const double* Vp;
  const double* z;
  const double* Bz;
  const double* D_in;
  double* c0_out;  // n
  double* Rv_out;  // n * m_v
  // stored closure factors: build writes, the VIF gradient pass reads (per row:
  // packed lower KS x KS factor, then 32 reciprocal pivots)
  double* Lfac_out;
  const double* Lfac_in;
  const double* A_in;
  const double* Ga_in;  // optional: Ga from the tiled SDDMM (tiles.cu tile_ga), n x 32, self at 31
  // Vecchia gradient in two passes: the factor pass writes each row's pair weights here (a~, w~ per
  // slot, c_d, c_u, w_d; kPairW doubles per row) and vecchia_pair_grad_kernel runs the pair loop
  double* pairw;
};
constexpr int kPairW = 68;

template <int KS>
constexpr int lfac_stride() {
  return KS * (KS + 1) / 2 + 32;
}

enum RowMode { kModeBuild = 0, kModeNll = 1, kModeGrad = 2, kModeVifGrad = 3 };

// The Vecchia gradient mode evaluates its closure covariances with the branch-free sqrt / exp
// (gneiting_eval_bf, ~ulp from the correctly rounded path); compile with -DSTGP_FAST_COV=0 for the
// correctly rounded covariances there too.
#ifndef STGP_FAST_COV
#define STGP_FAST_COV 1
#endif
__device__ __forceinline__ constexpr bool fast_cov() { return STGP_FAST_COV != 0; }

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Next row (schedule index) for this warp: a grid-stride step, or -- with a.next -- the next
// unclaimed row, so the rows in flight stay a contiguous window of the schedule whatever the
// per-row cost variations (L2 reuse of the gathered W columns).
__device__ __forceinline__ int next_row(const RowArgs& a, int static_next, int lane) {
  if (!a.next) return static_next;
  int c = 0;
  if (lane == 0) c = static_cast<int>(atomicAdd(a.next, 1ull));
  return __shfl_sync(0xffffffffu, c, 0);
}

// Per-row reduction contribution (lane 0): into the per-row slot when a.row_part is set
// (deterministic under dynamic claiming), else into the warp's running total.
__device__ __forceinline__ void row_acc(const RowArgs& a, double* tot, int i, int q, double x) {
  if (a.row_part)
    a.row_part[static_cast<size_t>(i - a.row_begin) * 8 + q] = x;
  else
    tot[q] += x;
}

// Closure Gram G = W_cl^T W_cl over 32 slots (lower 8x8 tiles, mirrored) with
// DMMA; scol[c] = column of slot c or -1.  Result into sG (row stride LD).
// WITH_X: also Ga[c] = W_{cl_c} . x (x = X(:, i)) as a fifth DMMA column block.
template <int LD, bool WITH_X>
__device__ __forceinline__ void closure_gram_dmma(const double* __restrict__ W, int ldw, const int* scol,
                                                  double* sG, int lane, const double* __restrict__ xcol,
                                                  double* sGa, const double* __restrict__ zcol) {
  const int grp = lane >> 2, tig = lane & 3;
  double acc[10][2];
  double accx[4][2];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int t = 0; t < 4; ++t) accx[t][0] = accx[t][1] = 0.0;
  const double* colp[4];
#pragma unroll
  for (int I = 0; I < 4; ++I) {
    const int c = scol[8 * I + grp];
    colp[I] = (c >= 0 ? W + static_cast<size_t>(c) * ldw : zcol) + tig;
  }
  const double* px = WITH_X ? xcol + tig : zcol + tig;
  // software pipelined: the next k-step's fragments are in flight while this step's DMMAs issue
  // (L2-latency bound otherwise); empty slots read the zero column, so the loads carry no
  // predicates.  ldw is a multiple of 8.
  double f[4], bx = 0.0;
#pragma unroll
  for (int I = 0; I < 4; ++I) f[I] = __ldg(colp[I]);
  if (WITH_X) bx = __ldg(px);
  auto step = [&](const double* fa, double xb) {
    if (WITH_X) {
      const double b = grp == 0 ? xb : 0.0;
#pragma unroll
      for (int I = 0; I < 4; ++I) dmma_f64(accx[I][0], accx[I][1], fa[I], b);
    }
    int t = 0;
#pragma unroll
    for (int I = 0; I < 4; ++I)
#pragma unroll
      for (int J = 0; J <= I; ++J) {
        dmma_f64(acc[t][0], acc[t][1], fa[I], fa[J]);
        ++t;
      }
  };
#pragma unroll 4
  for (int kb = 4; kb < ldw; kb += 4) {
    double fn[4], bxn = 0.0;
#pragma unroll
    for (int I = 0; I < 4; ++I) fn[I] = __ldg(colp[I] + kb);
    if (WITH_X) bxn = __ldg(px + kb);
    step(f, bx);
#pragma unroll
    for (int I = 0; I < 4; ++I) f[I] = fn[I];
    bx = bxn;
  }
  step(f, bx);
  int t = 0;
#pragma unroll
  for (int I = 0; I < 4; ++I)
#pragma unroll
    for (int J = 0; J <= I; ++J) {
      const int r = 8 * I + grp, c = 8 * J + 2 * tig;
      sG[r * LD + c] = acc[t][0];
      sG[r * LD + c + 1] = acc[t][1];
      sG[c * LD + r] = acc[t][0];
      sG[(c + 1) * LD + r] = acc[t][1];
      ++t;
    }
  if (WITH_X && tig == 0)
#pragma unroll
    for (int I = 0; I < 4; ++I) sGa[8 * I + grp] = accx[I][0];
}

// Time classes of a row's closure (its slots span few distinct times: same and previous time
// blocks).  Fills cls[lane] (class of slot `lane`) and the per-class-pair temporal factors of the
// lag table into tf[nc * nc]; returns nc, or 0 when more than kMaxCls classes (use the table).
constexpr int kMaxCls = 4;
__device__ __forceinline__ int closure_time_classes(const LagTable& lt, int pt, int myt, int lane, int* cls,
                                                    int* ctid, TF* tf) {
  const int key = pt >= 0 ? myt : -1;
  const unsigned same = __match_any_sync(kFull, key);
  const int leader = __ffs(same) - 1;
  const unsigned leaders = __ballot_sync(kFull, lane == leader && pt >= 0);
  const int nc = __popc(leaders);
  if (nc > kMaxCls) return 0;
  cls[lane] = __popc(leaders & ((1u << leader) - 1));
  if (lane == leader && pt >= 0) ctid[__popc(leaders & ((1u << lane) - 1))] = myt;
  __syncwarp();
  if (lane < nc * nc) tf[lane] = lt.get(ctid[lane / nc], ctid[lane % nc]);
  __syncwarp();
  return nc;
}

template <int MODE, bool HAS_W, int KS, bool GEN = false>  // GEN: general-nu covariances (value modes)
__global__ void __launch_bounds__(kRowWarps * 32, 4) vecchia_rows_kernel(RowArgs a) {
  static_assert(KS >= 1 && KS <= 31, "closure must fit a warp");
  constexpr int NS = KS + 1;           // closure slots
  constexpr int LD = 33;               // smem row stride (doubles)
  constexpr int NP = NS * (NS - 1) / 2;
  __shared__ uint16_t sPair[NP];
  __shared__ double sC[kRowWarps][32 * LD];
  __shared__ double sx[kRowWarps][32], sy[kRowWarps][32], sAw[kRowWarps][2][32];
  __shared__ double sCol[kRowWarps][2][32];
  __shared__ int st[kRowWarps][32], scol[kRowWarps][32];
  __shared__ double sred[kRowWarps][8];
  __shared__ TF stf[kRowWarps][kMaxCls * kMaxCls];
  __shared__ int scls[kRowWarps][32], sctid[kRowWarps][kMaxCls];

  for (int p = threadIdx.x; p < NP; p += blockDim.x) {
    int aa = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(p))) * 0.5f);
    while (aa * (aa - 1) / 2 > p) --aa;
    while ((aa + 1) * aa / 2 <= p) ++aa;
    sPair[p] = static_cast<uint16_t>(aa | ((p - aa * (aa - 1) / 2) << 8));
  }
  __syncthreads();

  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* C = sC[w];
  double tot[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) tot[q] = 0.0;

  const int gw = blockIdx.x * kRowWarps + w, nw = gridDim.x * kRowWarps;
  const int nrows = a.row_end - a.row_begin;
  for (int kr = next_row(a, gw, lane); kr < nrows; kr = next_row(a, kr + nw, lane)) {
    const int i = a.order ? __ldg(&a.order[kr]) : a.row_begin + kr;
    // ---- closure slots ----
    int nb = -1;
    if (lane < a.m_v) nb = __ldg(&a.nbr[static_cast<size_t>(i) * a.m_v + lane]);
    const int k = __popc(__ballot_sync(kFull, nb >= 0));  // neighbours packed at the front
    STGP_DCHECK(k <= KS);
    const int pt = lane < k ? nb : (lane == KS ? i : -1);
    double rp = 0.0, zp = 0.0;
    if (pt >= 0) {
      sx[w][lane] = __ldg(&a.x[pt]);
      sy[w][lane] = __ldg(&a.y[pt]);
      st[w][lane] = __ldg(&a.tid[pt]);
      if (MODE != kModeBuild) rp = __ldg(&a.r[pt]);
      if (MODE == kModeVifGrad) zp = __ldg(&a.z[pt]);
    }
    scol[w][lane] = pt;
    __syncwarp();
    const int nc = closure_time_classes(a.lt, pt, pt >= 0 ? st[w][lane] : -1, lane, scls[w], sctid[w], stf[w]);
    // VIF gradient: Ga[s] = W_{cl_s} . X_i (= U_{cl_s} . Hhat_i) from the same DMMA pass
    if (HAS_W)
      closure_gram_dmma<LD, MODE == kModeVifGrad>(a.W, a.ldw, scol[w], C, lane,
                                                 MODE == kModeVifGrad ? a.X + static_cast<size_t>(i) * a.ldw : nullptr,
                                                 sAw[w][0], a.zcol);  // Gram staged in C
    __syncwarp();
    double Ga = 0.0, aGa = 0.0;
    if (MODE == kModeVifGrad) {
      const double* xi = a.X + static_cast<size_t>(i) * a.ldw;
      Ga = pt >= 0 ? sAw[w][0][lane] : 0.0;
      const double* vi = a.Vp + static_cast<size_t>(i) * a.ldw;
      for (int j = lane; j < a.ldw; j += 32) aGa = fma(__ldg(&vi[j]), __ldg(&xi[j]), aGa);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) aGa += __shfl_xor_sync(kFull, aGa, o);
    }
    // ---- phase A: covariances over the closure (compact slot k maps to KS) ----
    const int P = (k + 1) * k / 2;
    auto slots = [&](int p, int& sa, int& sb) {
      STGP_DCHECK(p < NP);
      const int pr = sPair[p];
      const int ca = pr & 0xff;
      sb = pr >> 8;
      sa = ca == k ? KS : ca;
      STGP_DCHECK(sa < NS && sb < sa);
    };
    for (int p = lane; p < P; p += 32) {
      int sa, sb;
      slots(p, sa, sb);
      double pe, pb;
      if (nc) {
        const TF& fc = stf[w][scls[w][sa] * nc + scls[w][sb]];
        pe = fc.pow_mE;
        pb = fc.pow_mbh;
      } else {
        a.lt.get2(st[w][sa], st[w][sb], pe, pb);
      }
      TF f;
      f.pow_mE = pe;
      f.pow_mbh = pb;
      double v;
      if (MODE == kModeGrad && fast_cov()) {
        // likelihood-gradient evaluations (1e-8 parity): the branch-free sqrt / exp of the pair gradient
        const double dx = sx[w][sa] - sx[w][sb], dy = sy[w][sa] - sy[w][sb];
        v = gneiting_eval_bf(a.k, matern_poly(a.k.nu_code), fma(dx, dx, dy * dy), f);
      } else {
        v = gneiting_eval<GEN>(a.k, spatial_dist(sx[w][sa], sy[w][sa], sx[w][sb], sy[w][sb]), f);
      }
      if (HAS_W) v = __dsub_rn(v, C[sa * LD + sb]);  // each pair slot is owned by one lane
      C[sa * LD + sb] = v;
      C[sb * LD + sa] = v;
    }
    if (lane < k || lane == KS) {
      // diagonal: k(p,p) = sigma1_2 exactly; minus |w_p|^2 for VIF; plus nugget
      double v = a.s1;
      if (HAS_W) v = __dsub_rn(v, C[lane * LD + lane]);
      C[lane * LD + lane] = __dadd_rn(v, a.nugget);
    }
    __syncwarp();
    const double dii = C[KS * LD + KS];
    const double cval = lane < k ? C[KS * LD + lane] : 0.0;
    // ---- phase B: Cholesky of the KS x KS block (identity-padded) in registers ----
    double R[KS];
    double dinv = 0.0;  // lane j keeps 1 / L_jj
    bool ok = false;
    // the jitter ladder stays a rolled loop: unrolling it would triple the factorisation's code
#pragma unroll 1
    for (int attempt = 0; attempt < 3 && !ok; ++attempt) {
#pragma unroll
      for (int c = 0; c < KS; ++c) R[c] = (lane < k && c < k) ? C[lane * LD + c] : (c == lane ? 1.0 : 0.0);
      if (attempt >= 1 && lane < k) {
        // cumulative ladder: (C + j) then (C + j) + 9j, as the reference mutates C_N in place
        double d = __dadd_rn(C[lane * LD + lane], 1e-10 * a.s1);
        if (attempt == 2) d = __dadd_rn(d, 9.0 * (1e-10 * a.s1));
#pragma unroll
        for (int c = 0; c < KS; ++c)
          if (c == lane) R[c] = d;
      }
      bool good = true;
#pragma unroll
      for (int j = 0; j < KS; ++j) {
        const double piv = __shfl_sync(kFull, R[j], j);
        good = good && (piv > 0.0);
        const double inv = rsqrt(piv);
        R[j] = lane == j ? piv * inv : R[j] * inv;
        if (lane == j) dinv = inv;
        double* col = sCol[w][j & 1];
        col[lane] = R[j];
        __syncwarp();
#pragma unroll
        for (int c = j + 1; c < KS; ++c) R[c] = fma(-R[j], col[c], R[c]);  // upper entries: unused garbage
      }
      ok = __all_sync(kFull, good);
    }
    if (!ok) {
      if (lane == 0) atomicMin(a.fail_row, i);
      continue;
    }
    // L rows to smem for the back substitution (C no longer needed)
    __syncwarp();
#pragma unroll
    for (int c = 0; c < KS; ++c)
      if (c <= lane) C[lane * LD + c] = R[c];
    if (MODE == kModeBuild && a.Lfac_out && lane < KS) {
      double* dst = a.Lfac_out + static_cast<size_t>(i) * lfac_stride<KS>();
      const int off = lane * (lane + 1) / 2;
#pragma unroll
      for (int c = 0; c < KS; ++c)
        if (c <= lane) dst[off + c] = R[c];
      dst[KS * (KS + 1) / 2 + lane] = dinv;
    }
    __syncwarp();
    // ---- solves: b1 = C^{-1} c (A), b2 = C^{-1} r_N (gradient) ----
    constexpr bool TWO = (MODE == kModeGrad || MODE == kModeVifGrad);
    double Dst = 0.0, uz = 0.0;
    if (MODE == kModeVifGrad) {
      Dst = __ldg(&a.D_in[i]);
      uz = __ldg(&a.Bz[i]);
    }
    double b1 = cval;
    double b2 = 0.0;
    if (MODE == kModeGrad && lane < k) b2 = rp;
    if (MODE == kModeVifGrad && lane < k) b2 = (Ga + uz * zp) / Dst;  // vrow_N
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      if (lane == j) {
        b1 *= dinv;
        if (TWO) b2 *= dinv;
      }
      const double y1 = __shfl_sync(kFull, b1, j);
      const double y2 = TWO ? __shfl_sync(kFull, b2, j) : 0.0;
      if (lane > j) {
        b1 = fma(-R[j], y1, b1);
        if (TWO) b2 = fma(-R[j], y2, b2);
      }
    }
#pragma unroll
    for (int j = KS - 1; j >= 0; --j) {
      if (lane == j) {
        b1 *= dinv;
        if (TWO) b2 *= dinv;
      }
      const double x1 = __shfl_sync(kFull, b1, j);
      const double x2 = TWO ? __shfl_sync(kFull, b2, j) : 0.0;
      if (lane < j) {
        const double ljl = C[j * LD + lane];
        b1 = fma(-ljl, x1, b1);
        if (TWO) b2 = fma(-ljl, x2, b2);
      }
    }
    const double Aval = lane < k ? b1 : 0.0;
    const double wval = (TWO && lane < k) ? b2 : 0.0;  // C^{-1} r_N (Vecchia) or Rv (VIF)
    // ---- phase C: D, u ----
    double ac = Aval * cval, ar = Aval * (lane < k ? rp : 0.0), aa = Aval * Aval, aw = Aval * wval;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ac += __shfl_xor_sync(kFull, ac, o);
      if (MODE != kModeBuild) ar += __shfl_xor_sync(kFull, ar, o);
      if (TWO) {
        aa += __shfl_xor_sync(kFull, aa, o);
        aw += __shfl_xor_sync(kFull, aw, o);
      }
    }
    const double D = dii - ac;
    if (!(D > 0.0)) {
      if (lane == 0) atomicMin(a.fail_row, i);
      continue;
    }
    if (a.A_out && lane < a.m_v) a.A_out[static_cast<size_t>(i) * a.m_v + lane] = Aval;
    if (a.D_out && lane == 0) a.D_out[i] = D;
    if (MODE == kModeBuild) continue;
    const double ri = __shfl_sync(kFull, rp, KS);
    const double u = ri - ar;
    if (a.u_out && lane == 0) a.u_out[i] = u;
    if (lane == 0) row_acc(a, tot, i, 0, log(D) + u * u / D);
    if (!TWO) continue;
    if (MODE == kModeGrad && a.pairw) {  // two-pass gradient: hand the pair weights to the pair kernel
      double* pw = a.pairw + static_cast<size_t>(i) * kPairW;
      pw[lane] = lane < k ? -Aval : (lane == KS ? 1.0 : 0.0);
      pw[32 + lane] = wval;
      const double cd = 0.5 * (1.0 / D - u * u / (D * D)), cu = u / D;
      const double s1n = 1.0 + aa, s2n = -aw;
      const double wd = cd * s1n - cu * s2n;
      if (lane == 0) {
        pw[64] = cd;
        pw[65] = cu;
        pw[66] = wd;
        row_acc(a, tot, i, 1, wd);
      }
      continue;
    }
    // ---- phase D: gradient over closure pairs ----
    sAw[w][0][lane] = lane < k ? -Aval : (lane == KS ? 1.0 : 0.0);  // a~
    sAw[w][1][lane] = wval;                                          // w~ or Rv (0 at i)
    __syncwarp();
    double cd, cu;
    if (MODE == kModeVifGrad) {
      // Phi_i = c0 a~a~' - sym(a~ Rv')   (approximations.cpp:646-661)
      cd = 0.5 * (1.0 / Dst - (aGa + uz * uz) / (Dst * Dst));
      cu = 1.0;
      if (lane == 0) a.c0_out[i] = cd;
      if (lane < a.m_v) a.Rv_out[static_cast<size_t>(i) * a.m_v + lane] = wval;
    } else {
      cd = 0.5 * (1.0 / D - u * u / (D * D));
      cu = u / D;
    }
    // Branch-free pair gradient (gneiting_grad_bf: no special-case paths in sqrt / exp / Matern), the
    // class-table and lag-table variants as separate loops (nc is row-uniform).  A/B on one B200 at
    // cfg4: 14.49 -> 13.95 ms; two pairs per step (ILP) and an approximate-rsqrt Cholesky were slower.
    double g[6] = {0, 0, 0, 0, 0, 0};
    const MaternPoly mpol = matern_poly(a.k.nu_code);
    auto sq_dist = [&](int sa, int sb) {
      const double dx = sx[w][sa] - sx[w][sb], dy = sy[w][sa] - sy[w][sb];
      return fma(dx, dx, dy * dy);
    };
    auto weight = [&](int sa, int sb) {
      const double ta = sAw[w][0][sa], tb = sAw[w][0][sb], wa = sAw[w][1][sa], wb = sAw[w][1][sb];
      return cd * (2.0 * ta * tb) - cu * (wa * tb + wb * ta);
    };
    auto one_pair = [&](int sa, int sb, const TF& f) {
      double kg[6];
      gneiting_grad_bf(a.k, mpol, a.inv_c, sq_dist(sa, sb), f, kg);
      const double wt = weight(sa, sb);
#pragma unroll
      for (int q = 0; q < 6; ++q) g[q] = fma(wt, kg[q], g[q]);
    };
    if (nc) {
      for (int p = lane; p < P; p += 32) {
        int sa, sb;
        slots(p, sa, sb);
        STGP_DCHECK(scls[w][sa] < nc && scls[w][sb] < nc);
        one_pair(sa, sb, stf[w][scls[w][sa] * nc + scls[w][sb]]);
      }
    } else {
      for (int p = lane; p < P; p += 32) {
        int sa, sb;
        slots(p, sa, sb);
        one_pair(sa, sb, a.lt.get(st[w][sa], st[w][sb]));
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g[q] += __shfl_xor_sync(kFull, g[q], o);
    // diagonal pairs and the nugget slot: weight c_d * s1n - c_u * s2n
    const double s1n = 1.0 + aa, s2n = -aw;
    const double wd = cd * s1n - cu * s2n;
    if (lane == 0) {
      row_acc(a, tot, i, 1, wd);
#pragma unroll
      for (int q = 0; q < 6; ++q) row_acc(a, tot, i, 2 + q, g[q] + wd * a.g00[q]);
    }
    __syncwarp();
  }
  // deterministic block reduction: warps in order
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) sred[w][q] = tot[q];
  __syncthreads();
  if (threadIdx.x < 8) {
    double s = 0.0;
    for (int ww = 0; ww < kRowWarps; ++ww) s += sred[ww][threadIdx.x];
    a.part[static_cast<size_t>(blockIdx.x) * 8 + threadIdx.x] = s;
  }
}

// Second pass of the two-pass Vecchia gradient: the closure-pair loop of phase D above with the pair
// weights the factor pass stored (same pair order, arithmetic and per-row sums), at the occupancy of a
// kernel without the register Cholesky.  Per-block partials of q = 2..7 into a.part.
#ifndef STGP_PAIR_MINB
#define STGP_PAIR_MINB 7  // resident blocks per SM the pair kernel is compiled for (72 registers; 6: 12.92, 7: 12.85, 8: 12.89 ms)
#endif
template <int KS>
__global__ void __launch_bounds__(kRowWarps * 32, STGP_PAIR_MINB) vecchia_pair_grad_kernel(RowArgs a) {
  constexpr int NS = KS + 1;
  constexpr int NP = NS * (NS - 1) / 2;
  __shared__ uint16_t sPair[NP];
  __shared__ double sx[kRowWarps][32], sy[kRowWarps][32], sAw[kRowWarps][2][32];
  __shared__ int st[kRowWarps][32];
  __shared__ double sred[kRowWarps][8];
  __shared__ TF stf[kRowWarps][kMaxCls * kMaxCls];
  __shared__ int scls[kRowWarps][32], sctid[kRowWarps][kMaxCls];
  for (int p = threadIdx.x; p < NP; p += blockDim.x) {
    int aa = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(p))) * 0.5f);
    while (aa * (aa - 1) / 2 > p) --aa;
    while ((aa + 1) * aa / 2 <= p) ++aa;
    sPair[p] = static_cast<uint16_t>(aa | ((p - aa * (aa - 1) / 2) << 8));
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double tot[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) tot[q] = 0.0;
  const MaternPoly mpol = matern_poly(a.k.nu_code);
  const int gw = blockIdx.x * kRowWarps + w, nw = gridDim.x * kRowWarps;
  const int nrows = a.row_end - a.row_begin;
  for (int kr = gw; kr < nrows; kr += nw) {
    const int i = a.order ? __ldg(&a.order[kr]) : a.row_begin + kr;
    int nb = -1;
    if (lane < a.m_v) nb = __ldg(&a.nbr[static_cast<size_t>(i) * a.m_v + lane]);
    const int k = __popc(__ballot_sync(kFull, nb >= 0));
    const int pt = lane < k ? nb : (lane == KS ? i : -1);
    if (pt >= 0) {
      sx[w][lane] = __ldg(&a.x[pt]);
      sy[w][lane] = __ldg(&a.y[pt]);
      st[w][lane] = __ldg(&a.tid[pt]);
    }
    const double* pw = a.pairw + static_cast<size_t>(i) * kPairW;
    sAw[w][0][lane] = __ldg(&pw[lane]);
    sAw[w][1][lane] = __ldg(&pw[32 + lane]);
    const double cd = __ldg(&pw[64]), cu = __ldg(&pw[65]), wd = __ldg(&pw[66]);
    __syncwarp();
    const int nc = closure_time_classes(a.lt, pt, pt >= 0 ? st[w][lane] : -1, lane, scls[w], sctid[w], stf[w]);
    const int P = (k + 1) * k / 2;
    auto slots = [&](int p, int& sa, int& sb) {
      const int pr = sPair[p];
      const int ca = pr & 0xff;
      sb = pr >> 8;
      sa = ca == k ? KS : ca;
    };
    double g[6] = {0, 0, 0, 0, 0, 0};
    auto one_pair = [&](int sa, int sb, const TF& f) {
      const double dx = sx[w][sa] - sx[w][sb], dy = sy[w][sa] - sy[w][sb];
      double kg[6];
      gneiting_grad_bf(a.k, mpol, a.inv_c, fma(dx, dx, dy * dy), f, kg);
      const double ta = sAw[w][0][sa], tb = sAw[w][0][sb], wa = sAw[w][1][sa], wb = sAw[w][1][sb];
      const double wt = cd * (2.0 * ta * tb) - cu * (wa * tb + wb * ta);
#pragma unroll
      for (int q = 0; q < 6; ++q) g[q] = fma(wt, kg[q], g[q]);
    };
    if (nc) {
      for (int p = lane; p < P; p += 32) {
        int sa, sb;
        slots(p, sa, sb);
        one_pair(sa, sb, stf[w][scls[w][sa] * nc + scls[w][sb]]);
      }
    } else {
      for (int p = lane; p < P; p += 32) {
        int sa, sb;
        slots(p, sa, sb);
        one_pair(sa, sb, a.lt.get(st[w][sa], st[w][sb]));
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g[q] += __shfl_xor_sync(kFull, g[q], o);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 6; ++q) tot[2 + q] += g[q] + wd * a.g00[q];
    __syncwarp();
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) sred[w][q] = tot[q];
  __syncthreads();
  if (threadIdx.x < 8) {
    double s = 0.0;
    for (int ww = 0; ww < kRowWarps; ++ww) s += sred[ww][threadIdx.x];
    a.part[static_cast<size_t>(blockIdx.x) * 8 + threadIdx.x] = s;
  }
}

// Ga[s] = W_{cl_s} . x for the 32 closure slots (4 DMMA blocks per k-step).
__device__ __forceinline__ void closure_x_dmma(const double* __restrict__ W, int ldw, const int* scol,
                                               const double* __restrict__ xcol, double* sGa, int lane,
                                               const double* __restrict__ zcol) {
  const int grp = lane >> 2, tig = lane & 3;
  double accx[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) accx[t][0] = accx[t][1] = 0.0;
  const double* colp[4];
#pragma unroll
  for (int I = 0; I < 4; ++I) {
    const int c = scol[8 * I + grp];
    colp[I] = (c >= 0 ? W + static_cast<size_t>(c) * ldw : zcol) + tig;
  }
  const double* px = xcol + tig;
  // two k-steps of fragments in flight (L2-latency bound otherwise); no load predicates (empty
  // slots read the zero column); ldw is a multiple of 8
  double f0[4], f1[4], x0, x1;
#pragma unroll
  for (int I = 0; I < 4; ++I) {
    f0[I] = __ldg(colp[I]);
    f1[I] = __ldg(colp[I] + 4);
  }
  x0 = __ldg(px);
  x1 = __ldg(px + 4);
  auto step = [&](const double* fa, double xb) {
    const double b = grp == 0 ? xb : 0.0;
#pragma unroll
    for (int I = 0; I < 4; ++I) dmma_f64(accx[I][0], accx[I][1], fa[I], b);
  };
#pragma unroll 4
  for (int kb = 8; kb < ldw; kb += 4) {
    double fn[4];
#pragma unroll
    for (int I = 0; I < 4; ++I) fn[I] = __ldg(colp[I] + kb);
    const double xn = __ldg(px + kb);
    step(f0, x0);
#pragma unroll
    for (int I = 0; I < 4; ++I) {
      f0[I] = f1[I];
      f1[I] = fn[I];
    }
    x0 = x1;
    x1 = xn;
  }
  step(f0, x0);
  step(f1, x1);
  if (tig == 0)
#pragma unroll
    for (int I = 0; I < 4; ++I) sGa[8 * I + grp] = accx[I][0];
}

// VIF gradient rows from the build's stored factors (approximations.cpp:616-697):
// Ga, aGa, vrow, Rv = C_N^{-1} vrow_N with the stored Cholesky factor, c0, Phi_i
// weights and the direct-pass kernel gradients.  No Gram, assembly or factorisation.
template <int KS>
__global__ void __launch_bounds__(kRowWarps * 32) vif_grad_stored_kernel(RowArgs a) {
  constexpr int NS = KS + 1;
  constexpr int LD = 33;
  constexpr int NP = NS * (NS - 1) / 2;
  __shared__ uint16_t sPair[NP];
  __shared__ double sL[kRowWarps][32 * LD];
  __shared__ double sx[kRowWarps][32], sy[kRowWarps][32], sAw[kRowWarps][2][32], sGa[kRowWarps][32];
  __shared__ int st[kRowWarps][32], scol[kRowWarps][32];
  __shared__ double sred[kRowWarps][8];
  // per-row cache of the temporal factors of the closure's time classes (a row's closure spans a
  // few distinct times: the KG loop then reads TF from shared memory instead of two dependent
  // global lookups per pair)
  __shared__ TF stf[kRowWarps][kMaxCls * kMaxCls];
  __shared__ int scls[kRowWarps][32], sctid[kRowWarps][kMaxCls];
  for (int p = threadIdx.x; p < NP; p += blockDim.x) {
    int aa = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(p))) * 0.5f);
    while (aa * (aa - 1) / 2 > p) --aa;
    while ((aa + 1) * aa / 2 <= p) ++aa;
    sPair[p] = static_cast<uint16_t>(aa | ((p - aa * (aa - 1) / 2) << 8));
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* Lw = sL[w];
  double tot[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) tot[q] = 0.0;
  const int gw = blockIdx.x * kRowWarps + w, nw = gridDim.x * kRowWarps;
  const int nrows = a.row_end - a.row_begin;
  for (int kr = next_row(a, gw, lane); kr < nrows; kr = next_row(a, kr + nw, lane)) {
    const int i = a.order ? __ldg(&a.order[kr]) : a.row_begin + kr;
    int nb = -1;
    if (lane < a.m_v) nb = __ldg(&a.nbr[static_cast<size_t>(i) * a.m_v + lane]);
    const int k = __popc(__ballot_sync(kFull, nb >= 0));
    const int pt = lane < k ? nb : (lane == KS ? i : -1);
    double zp = 0.0;
    if (pt >= 0) {
      sx[w][lane] = __ldg(&a.x[pt]);
      sy[w][lane] = __ldg(&a.y[pt]);
      st[w][lane] = __ldg(&a.tid[pt]);
      zp = __ldg(&a.z[pt]);
    }
    scol[w][lane] = pt;
    __syncwarp();
    if (a.Ga_in) {
      const double* gi = a.Ga_in + static_cast<size_t>(i) * 32;
      sGa[w][lane] = lane < k ? __ldg(&gi[lane]) : (lane == KS ? __ldg(&gi[31]) : 0.0);
    } else {
      closure_x_dmma(a.W, a.ldw, scol[w], a.X + static_cast<size_t>(i) * a.ldw, sGa[w], lane, a.zcol);
    }
    // stored factor: row `lane` of L into registers and shared memory
    const double* src = a.Lfac_in + static_cast<size_t>(i) * lfac_stride<KS>();
    double R[KS];
    const int off = lane * (lane + 1) / 2;
#pragma unroll
    for (int c = 0; c < KS; ++c) R[c] = (lane < KS && c <= lane) ? __ldg(&src[off + c]) : 0.0;
    const double dinv = lane < KS ? __ldg(&src[KS * (KS + 1) / 2 + lane]) : 0.0;
#pragma unroll
    for (int c = 0; c < KS; ++c)
      if (c <= lane && lane < KS) Lw[lane * LD + c] = R[c];
    __syncwarp();
    const double Dst = __ldg(&a.D_in[i]), uz = __ldg(&a.Bz[i]);
    const double Ga = pt >= 0 ? sGa[w][lane] : 0.0;
    double b2 = lane < k ? (Ga + uz * zp) / Dst : 0.0;  // vrow_N
#pragma unroll
    for (int j = 0; j < KS; ++j) {
      if (lane == j) b2 *= dinv;
      const double y2 = __shfl_sync(kFull, b2, j);
      if (lane > j) b2 = fma(-R[j], y2, b2);
    }
#pragma unroll
    for (int j = KS - 1; j >= 0; --j) {
      if (lane == j) b2 *= dinv;
      const double x2 = __shfl_sync(kFull, b2, j);
      if (lane < j) b2 = fma(-Lw[j * LD + lane], x2, b2);
    }
    const double Rv = lane < k ? b2 : 0.0;
    const double Aval = lane < k ? __ldg(&a.A_in[static_cast<size_t>(i) * a.m_v + lane]) : 0.0;
    // aGa = V'_i . X_i = (W_i - sum_a A_ia W_{N_a}) . X_i = Ga[self] - sum_a A_ia Ga[a]: no pass over V'_i
    double aa = Aval * Aval, aw = Aval * Rv, ag = Aval * Ga;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      aa += __shfl_xor_sync(kFull, aa, o);
      aw += __shfl_xor_sync(kFull, aw, o);
      ag += __shfl_xor_sync(kFull, ag, o);
    }
    const double aGa = __shfl_sync(kFull, Ga, KS) - ag;
    const double cd = 0.5 * (1.0 / Dst - (aGa + uz * uz) / (Dst * Dst));  // c0
    if (lane == 0) a.c0_out[i] = cd;
    if (lane < a.m_v) a.Rv_out[static_cast<size_t>(i) * a.m_v + lane] = Rv;
    sAw[w][0][lane] = lane < k ? -Aval : (lane == KS ? 1.0 : 0.0);
    sAw[w][1][lane] = Rv;
    const int nc = closure_time_classes(a.lt, pt, pt >= 0 ? st[w][lane] : -1, lane, scls[w], sctid[w], stf[w]);
    const bool cached = nc > 0;
    const int P = (k + 1) * k / 2;
    double g[6] = {0, 0, 0, 0, 0, 0};
    const MaternPoly mpol = matern_poly(a.k.nu_code);
    auto one_pair = [&](int sa, int sb, const TF& f) {  // branch-free pair gradient (as vecchia_rows_kernel)
      const double dx = sx[w][sa] - sx[w][sb], dy = sy[w][sa] - sy[w][sb];
      double kg[6];
      gneiting_grad_bf(a.k, mpol, a.inv_c, fma(dx, dx, dy * dy), f, kg);
      const double ta = sAw[w][0][sa], tb = sAw[w][0][sb], wa = sAw[w][1][sa], wb = sAw[w][1][sb];
      const double wt = cd * (2.0 * ta * tb) - (wa * tb + wb * ta);
#pragma unroll
      for (int q = 0; q < 6; ++q) g[q] = fma(wt, kg[q], g[q]);
    };
    auto slots = [&](int p, int& sa, int& sb) {
      STGP_DCHECK(p < NP);
      const int pr = sPair[p];
      const int ca = pr & 0xff;
      sb = pr >> 8;
      sa = ca == k ? KS : ca;
      STGP_DCHECK(sa < NS && sb < sa);
    };
    if (cached) {
      for (int p = lane; p < P; p += 32) {
        int sa, sb;
        slots(p, sa, sb);
        STGP_DCHECK(scls[w][sa] < nc && scls[w][sb] < nc);
        one_pair(sa, sb, stf[w][scls[w][sa] * nc + scls[w][sb]]);
      }
    } else {
      for (int p = lane; p < P; p += 32) {
        int sa, sb;
        slots(p, sa, sb);
        one_pair(sa, sb, a.lt.get(st[w][sa], st[w][sb]));
      }
    }
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g[q] += __shfl_xor_sync(kFull, g[q], o);
    const double wd = cd * (1.0 + aa) - (-aw);
    if (lane == 0) {
      row_acc(a, tot, i, 1, wd);
#pragma unroll
      for (int q = 0; q < 6; ++q) row_acc(a, tot, i, 2 + q, g[q] + wd * a.g00[q]);
    }
    __syncwarp();
  }
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) sred[w][q] = tot[q];
  __syncthreads();
  if (threadIdx.x < 8) {
    double s2 = 0.0;
    for (int ww = 0; ww < kRowWarps; ++ww) s2 += sred[ww][threadIdx.x];
    a.part[static_cast<size_t>(blockIdx.x) * 8 + threadIdx.x] = s2;
  }
}

// Fixed-order reduction of per-row contributions: block b sums rows [b*chunk, (b+1)*chunk).
static __global__ void __launch_bounds__(256) row_part_reduce_kernel(const double* rp, int nrows, int chunk,
                                                                     double* part) {
  __shared__ double red[8][256];
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int r0 = blockIdx.x * chunk, r1 = min(nrows, r0 + chunk);
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x)
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] += rp[static_cast<size_t>(r) * 8 + q];
#pragma unroll
  for (int q = 0; q < 8; ++q) red[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o)
#pragma unroll
      for (int q = 0; q < 8; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 8) part[static_cast<size_t>(blockIdx.x) * 8 + threadIdx.x] = red[threadIdx.x][0];
}

// Sum per-block partials in a fixed order: out[q] = sum_b part[b][q] (compensated).
// Compensated (Kahan) sum of the per-block partials, one warp per column: lane l sums blocks l, l + 32,
// ... in order, then lane 0 sums the 32 lane sums and their compensations in lane order (fixed order:
// deterministic; the dependent add chain is 1/32 of the one-thread loop's).
static __global__ void reduce_parts_kernel(const double* part, int nblocks, int width, double* out) {
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (q >= width) return;
  double s = 0.0, c = 0.0;
  for (int b = lane; b < nblocks; b += 32) {
    const double y = part[static_cast<size_t>(b) * width + q] - c;
    const double t = s + y;
    c = (t - s) - y;
    s = t;
  }
  __shared__ double ls[8][32], lc[8][32];
  ls[q][lane] = s;
  lc[q][lane] = c;
  __syncwarp();
  if (lane == 0) {
    double S = 0.0, C = 0.0;
    for (int l = 0; l < 64; ++l) {
      const double y = (l < 32 ? ls[q][l] : -lc[q][l - 32]) - C;
      const double t = S + y;
      C = (t - S) - y;
      S = t;
    }
    out[q] = S;
  }
}

}  // namespace stgp

// FP64 GEMM on the INT8 tensor cores (Ozaki scheme I, error-free slicing).
//
// B200's FP64 pipes (DMMA and DFMA) peak at ~37 TFLOP/s, while its int8 tensor cores (tcgen05.mma
// kind::i8) run at several POPS.  An FP64 product
//   C[r][j] = sum_c A[r][c] B[j][c]            (rows of A and B contiguous over c)
// is computed exactly up to the slicing truncation:
//   * row r of A is scaled by 2^-eA[r] into (-1, 1) and cut into S int8 slices of 7 bits each,
//     a = sum_s A_s 2^-7s (every step exact in FP64); B likewise per row j;
//   * the products A_s B_t with s + t = d share the scale 2^-7d; the hand-written tcgen05 kernel
//     (ozaki_tc.cu) accumulates every diagonal d in its own TMEM block, exactly in int32
//     (|C_d| <= S k 127^2 < 2^31 for k < 2^31 / (S 127^2));
//   * C = 2^(eA + eB) sum_{d = 2}^{S + 1} 2^-7d C_d, summed in FP64 from the smallest term in the
//     kernel's epilogue (the int32 partials never reach HBM).
// Terms with s + t > S + 1 are dropped: the result carries ~7 S bits relative to
// max_c |A[r][c]| max_c |B[j][c]| k (S = 7: 49 bits; far below the 1e-8 parity tolerance of the
// evaluation, tests/test_gpu_ozaki.py measures it against exact dot products and the DMMA GEMM).

#include <fstream>
#include <string>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <memory>
#include <tuple>

#include "lowrank_common.cuh"
#include "ozaki.cuh"

namespace stgp {

namespace {

// The S base-128 digits of trunc(v 2^(7 S)) for |v| < 1 (v already scaled, exact): all digits carry
// the sign of v and lie in [-127, 127]; digit 1 is the most significant.  Same digits as the FP64
// recurrence w = 128 v, t = trunc(w), v = w - t, at one FP64 multiply, one conversion and 32-bit
// funnel shifts (S is a compile-time constant).
struct Fixed {
  unsigned lo, hi;
  int sg;  // 0 or -1
};
template <int S>
__device__ __forceinline__ Fixed fixed_point(double v) {
  const long long q = __double2ll_rz(v * static_cast<double>(1LL << (7 * S)));  // exact scaling, truncation
  const unsigned long long a = q < 0 ? static_cast<unsigned long long>(-q) : static_cast<unsigned long long>(q);
  return Fixed{static_cast<unsigned>(a), static_cast<unsigned>(a >> 32), q < 0 ? -1 : 0};
}
template <int S>
__device__ __forceinline__ int digit(const Fixed& f, int s) {
  const int sh = 7 * (S - s);
  const unsigned d = (sh >= 32 ? (f.hi >> (sh - 32)) : __funnelshift_r(f.lo, f.hi, sh)) & 127u;
  return (static_cast<int>(d) ^ f.sg) - f.sg;
}
__device__ __forceinline__ unsigned pack4(int a, int b, int c, int d) {  // low bytes of a, b, c, d
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// One warp per row: exponent of the row maximum (scale[r] = 2^e > max |row|), then the S slices
// (char4 stores).  reverse: slice t stored at (S - t) kp (B operand), else at (t - 1) kp.
template <int S>
__global__ void __launch_bounds__(256) slice_rows_kernel(long long nrows, int k, int kp, const double* __restrict__ A,
                                                         int lda, bool reverse, int8_t* __restrict__ out,
                                                         long long ldo, double* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  for (long long r = warp; r < nrows; r += nw) {
    const double* a = A + r * lda;
    double mx = 0.0;
    for (int c = lane; c < k; c += 32) mx = fmax(mx, fabs(a[c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (lane == 0) scale[r] = ldexp(1.0, e);
    const double inv = ldexp(1.0, -e);
    int8_t* o = out + r * ldo;
    for (int c4 = lane * 4; c4 < kp; c4 += 128) {  // kp: k padded to 16 (zero slices)
      Fixed q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = fixed_point<S>(c4 + u < k ? a[c4 + u] * inv : 0.0);  // exact scale
#pragma unroll
      for (int s = 1; s <= S; ++s)
        *reinterpret_cast<unsigned*>(o + (reverse ? (S - s) : (s - 1)) * kp + c4) =
            pack4(digit<S>(q[0], s), digit<S>(q[1], s), digit<S>(q[2], s), digit<S>(q[3], s));
    }
  }
}

// Column form (A m x n column-major, lda; column r optionally multiplied by colD[r]); the product
// runs over n in chunks of L.  A block covers 32 rows j (lanes: every load is a 256-byte row
// segment) and 8 x 32 columns r (warps); each thread keeps its 32 values of one row in registers.
constexpr int kSlCols = 256;  // columns r per block; L is a multiple

// per-(chunk, row) maxima: atomicMax on the bit patterns of non-negative doubles (order-preserving).
// A block takes 256 consecutive reduction rows r (one chunk: L is a multiple of 256) and walks the m
// product rows j in segments of 256: each warp reads its 32 rows r as 2 KB contiguous runs, so the
// column-major source streams through DRAM in whole pages (the 256-byte column pieces of a j-tiled
// walk ran at ~3.3 TB/s); warp partials meet in shared memory, one global atomic per (block, j).
constexpr int kMaxRowsPerBlock = 256;
__global__ void __launch_bounds__(256) colmax_rows_kernel(int m, long long n, int L, const double* __restrict__ A,
                                                          int lda, const double* __restrict__ colD,
                                                          unsigned long long* __restrict__ maxbits) {
  __shared__ double part[8][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long r0 = static_cast<long long>(blockIdx.x) * kMaxRowsPerBlock;
  const int c = static_cast<int>(r0 / L);
  for (int j0 = 0; j0 < m; j0 += 256) {
    double mx[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) mx[u] = 0.0;
    for (int q = 0; q < 32; ++q) {
      const long long r = r0 + w * 32 + q;
      if (r >= n) break;
      const double f = colD ? fabs(__ldg(&colD[r])) : 1.0;
      const double* row = A + r * lda + j0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = 32 * u + lane;
        if (j0 + j < m) mx[u] = fmax(mx[u], fabs(__ldg(&row[j])) * f);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) part[w][32 * u + lane] = mx[u];
    __syncthreads();
    {
      const int j = threadIdx.x;
      double v = part[0][j];
#pragma unroll
      for (int ww = 1; ww < 8; ++ww) v = fmax(v, part[ww][j]);
      if (j0 + j < m && v > 0.0) atomicMax(&maxbits[static_cast<size_t>(c) * m + j0 + j], __double_as_longlong(v));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) colmax_kernel(int m, long long n, int L, const double* __restrict__ A, int lda,
                                                     const double* __restrict__ colD,
                                                     unsigned long long* __restrict__ maxbits) {
  const long long rb = static_cast<long long>(blockIdx.x) * kSlCols + (threadIdx.x >> 5) * 32;
  const int j = blockIdx.y * 32 + (threadIdx.x & 31);
  const int c = static_cast<int>((static_cast<long long>(blockIdx.x) * kSlCols) / L);
  double mx = 0.0;
  if (j < m) {
#pragma unroll 8
    for (int u = 0; u < 32; ++u) {
      const long long r = rb + u;
      if (r < n) {
        const double a = A[r * lda + j];
        mx = fmax(mx, fabs(colD ? a * __ldg(&colD[r]) : a));
      }
    }
  }
  if (j < m && mx > 0.0) atomicMax(&maxbits[static_cast<size_t>(c) * m + j], __double_as_longlong(mx));
}

// Row j of chunk c is scaled by scale[c * m + j] = 2^e (> the chunk maximum) and sliced into
// out[((c * m + j) * S + s - 1) * L + rl] and/or out_rev[((c * m + j) * S + S - s) * L + rl].  The
// digits of the block's 32 rows x 256 columns are staged in shared memory and leave as 256-byte
// row runs (full sectors, no partial-sector write-backs).
template <int H>  // rows r per block = 128 H
constexpr int sl_row() { return 128 * H + 16; }  // staged row pitch (bytes): spreads the 16-byte stores over banks
template <int S, int H>
__global__ void __launch_bounds__(256) slice_cols_kernel(int m, long long n, int L, const double* __restrict__ A,
                                                         int lda, const double* __restrict__ colD,
                                                         const unsigned long long* __restrict__ maxbits,
                                                         int8_t* __restrict__ out, int8_t* __restrict__ out_rev,
                                                         double* __restrict__ scale, int jfast) {
  constexpr int kRB = 128 * H, kRow = sl_row<H>();
  extern __shared__ __align__(16) unsigned char sd[];  // S * 32 * kRow digit bytes, then kRB x 32 doubles
  double* sa = reinterpret_cast<double*>(sd + S * 32 * kRow);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // jfast: the 32-row segments j vary fastest over consecutive blocks (the resident blocks read whole
  // source rows r) instead of the row blocks
  const unsigned bx = jfast ? blockIdx.y : blockIdx.x, by = jfast ? blockIdx.x : blockIdx.y;
  const long long rc0 = static_cast<long long>(bx) * kRB;
  const long long rb = rc0 + w * 16 * H;
  const int j0 = by * 32, j = j0 + lane;
  const int c = static_cast<int>(rc0 / L);
  // the block's kRB x 32 source tile in flight at once: 16-byte cp.async pieces (two doubles; m is a
  // multiple of 4, so a piece is wholly inside or outside), zero-filled beyond n and m
  for (int e = threadIdx.x; e < kRB * 16; e += blockDim.x) {
    const int row = e >> 4, piece = e & 15;
    const long long r = rc0 + row;
    const int jj = j0 + 2 * piece;
    const bool ok = r < n && jj < m;
    const double* src = ok ? A + r * lda + jj : A;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sa + row * 32 + 2 * piece));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0));
  }
  asm volatile("cp.async.commit_group;\n" ::);
  double inv = 0.0;
  if (j < m) {
    const double mx = __longlong_as_double(static_cast<long long>(maxbits[static_cast<size_t>(c) * m + j]));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    if (rc0 % L == 0 && w == 0) scale[static_cast<size_t>(c) * m + j] = ldexp(1.0, e);
    inv = ldexp(1.0, -e);
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
#pragma unroll
  for (int h = 0; h < H; ++h) {
    Fixed q[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const long long r = rb + 16 * h + u;
      double v = 0.0;
      if (j < m && r < n) {
        const double a = sa[(r - rc0) * 32 + lane];
        v = (colD ? a * __ldg(&colD[r]) : a) * inv;  // exact power-of-two scale
      }
      q[u] = fixed_point<S>(v);
    }
#pragma unroll
    for (int s = 1; s <= S; ++s) {
      uint4 v4;
      v4.x = pack4(digit<S>(q[0], s), digit<S>(q[1], s), digit<S>(q[2], s), digit<S>(q[3], s));
      v4.y = pack4(digit<S>(q[4], s), digit<S>(q[5], s), digit<S>(q[6], s), digit<S>(q[7], s));
      v4.z = pack4(digit<S>(q[8], s), digit<S>(q[9], s), digit<S>(q[10], s), digit<S>(q[11], s));
      v4.w = pack4(digit<S>(q[12], s), digit<S>(q[13], s), digit<S>(q[14], s), digit<S>(q[15], s));
      *reinterpret_cast<uint4*>(sd + ((s - 1) * 32 + lane) * kRow + w * 16 * H + 16 * h) = v4;
    }
  }
  __syncthreads();
  // copy-out: kRB / 16 threads per (slice, row) run of kRB bytes
  constexpr int kPieces = kRB / 16;
  const size_t off = static_cast<size_t>(rc0 - static_cast<long long>(c) * L);
  for (int e = threadIdx.x; e < S * 32 * kPieces; e += blockDim.x) {
    const int row = e / kPieces, piece = e % kPieces;
    const int s = row / 32 + 1, jj = row - (s - 1) * 32;
    if (j0 + jj >= m) continue;
    const uint4 v4 = *reinterpret_cast<const uint4*>(sd + row * kRow + piece * 16);
    const size_t base = (static_cast<size_t>(c) * m + j0 + jj) * S * static_cast<size_t>(L) + off + piece * 16;
    if (out) *reinterpret_cast<uint4*>(out + base + static_cast<size_t>(s - 1) * L) = v4;
    if (out_rev) *reinterpret_cast<uint4*>(out_rev + base + static_cast<size_t>(S - s) * L) = v4;
  }
}

// dispatch on the slice count (compile-time shifts)
#define STGP_OZ_SWITCH(S_, CALL)                                                  \
  switch (S_) {                                                                   \
    case 2: { constexpr int kS = 2; CALL; } break;                                \
    case 3: { constexpr int kS = 3; CALL; } break;                                \
    case 4: { constexpr int kS = 4; CALL; } break;                                \
    case 5: { constexpr int kS = 5; CALL; } break;                                \
    case 6: { constexpr int kS = 6; CALL; } break;                                \
    case 7: { constexpr int kS = 7; CALL; } break;                                \
    case 8: { constexpr int kS = 8; CALL; } break;                                \
    default: throw Error(kConfig, "ozaki: STGP_OZAKI_S must lie in [2, 8]");   \
  }

__global__ void sqrt_vec_kernel(long long n, const double* __restrict__ d, double* __restrict__ f) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    f[i] = sqrt(d[i]);
}

__global__ void rsqrt_vec_kernel(long long n, const double* __restrict__ d, double* __restrict__ f) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    f[i] = 1.0 / sqrt(d[i]);  // the factor of lowrank.cu scale_cols_kernel
}

}  // namespace

struct OzakiState {
  OzakiTcState* tc = nullptr;  // the tcgen05 kernel's work lists
  DevBuf<int8_t> As, Bs;
  DevBuf<double> sA, sB, colf, colf2;
  DevBuf<double> Tt;  // transposed triangular factor (ozaki_trmm_left)
  DevBuf<int8_t> keep;  // forward digits of the last ozaki_syrk_keep operand (V' D^{-1/2})
  DevBuf<double> keep_s;
  uint64_t keep_tag = 0;
  int keep_m = 0;
  long long keep_n = 0;
  DevBuf<unsigned long long> maxbits;
  ~OzakiState() { ozaki_tc_release(tc); }
};

void ozaki_release(stgp_ctx* ctx) {
  delete ctx->ozaki;
  ctx->ozaki = nullptr;
}

// Slices per form: the long reductions (K = S S^T, V'F^T; STGP_OZAKI_S_COLS, default S) carry the
// error budget (cfg4, worst gradient component vs DMMA: 2.8e-11 at 7 slices, 3.1e-9 at 6); the row
// form (X = K^-1 V', FITC K^-1 W; STGP_OZAKI_S_ROWS) costs nothing measurable at 6 (3.4e-11 with
// the column products at 7; 1.6e-9 at 5), which saves a quarter of its int8 work.
static int slices_for(const char* var, int dflt) {
  const char* e = std::getenv(var);
  if (e) return std::max(2, std::min(8, std::atoi(e)));
  return std::getenv("STGP_OZAKI_S") ? ozaki_slices() : dflt;
}

int ozaki_slices() {
  static const int s = [] {
    const char* e = std::getenv("STGP_OZAKI_S");
    return std::max(2, std::min(8, e ? std::atoi(e) : 7));
  }();
  return s;
}

bool ozaki_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STGP_OZAKI");  // A/B switch: 0 = the DMMA GEMM
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

// The slicing and combine passes are O(n m) against the O(n m^2) products: below a few hundred
// inducing points the DMMA GEMM wins (cfg3, M = 180: 6.9 vs 10.0 ms per evaluation).
bool ozaki_for(int m) {
  static const int min_m = [] {
    const char* e = std::getenv("STGP_OZAKI_MIN_M");
    return e ? std::atoi(e) : 512;
  }();
  return ozaki_enabled() && m >= min_m;
}

static int slice_halves() {
  static const int h = [] {
    const char* e = std::getenv("STGP_OZ_SLICE_H");  // tuning switch: rows per slicing block = 128 H (1 or 2)
    return e && std::atoi(e) == 2 ? 2 : 1;
  }();
  return h;
}

static int slice_jfast() {
  static const int v = [] {
    // block order of the column slicer: j segments fastest (default; cfg4 evaluation 270.0 -> 268.5 ms
    // although the slicer itself takes the same 5.8 ms either way) or row blocks fastest (0)
    const char* e = std::getenv("STGP_OZ_SLICE_JFAST");
    return e && std::atoi(e) == 0 ? 0 : 1;
  }();
  return v;
}

static bool colmax_rows() {
  static const bool on = [] {
    const char* e = std::getenv("STGP_OZ_COLMAX_ROWS");  // A/B switch: 0 = the j-tiled colmax
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

static OzakiState* state(stgp_ctx* ctx) {
  if (!ctx->ozaki) ctx->ozaki = new OzakiState();
  return ctx->ozaki;
}

static void rows_product(stgp_ctx* ctx, int S, long long n, int m, int k, const double* A, int lda, const double* B,
                         int ldb, double* C, int ldc, int tri = 0) {
  if (n <= 0 || m <= 0) return;
  if (m % 4 || ldc % 4) config_error("ozaki_gemm_rows: m and ldc must be multiples of 4");
  const int kp = (k + 31) / 32 * 32;  // slice stride: whole 32-byte K steps of the tcgen05 kernel
  if (static_cast<long long>(S) * kp * 127 * 127 >= (1LL << 31)) config_error("ozaki: k too large for exact int32");
  OzakiState* oz = state(ctx);
  cudaStream_t st = ctx->stream;
  const int ldk = S * kp;
  // B slices (m rows, reversed slice order) and scales
  oz->Bs.ensure(static_cast<size_t>(m) * ldk);
  oz->sB.ensure(m);
  STGP_OZ_SWITCH(S, (slice_rows_kernel<kS><<<grid_for(static_cast<long long>(m) * 32, 256), 256, 0, st>>>(
                         m, k, kp, B, ldb, true, oz->Bs.get(), ldk, oz->sB.get())));
  launched(ctx);
  // no int32 partials leave the SM, so chunks only bound the digit buffer (~1.5 GB)
  const long long chunk = std::min<long long>(n, std::max<long long>(16384, (3LL << 29) / ldk));
  oz->As.ensure(static_cast<size_t>(chunk) * ldk);
  oz->sA.ensure(static_cast<size_t>(chunk));
  for (long long r0 = 0; r0 < n; r0 += chunk) {
    const long long nr = std::min(chunk, n - r0);
    STGP_OZ_SWITCH(S, (slice_rows_kernel<kS><<<grid_for(nr * 32, 256), 256, 0, st>>>(
                           nr, k, kp, A + r0 * lda, lda, false, oz->As.get(), ldk, oz->sA.get())));
    launched(ctx);
    ProfRegion pr(ctx, "oz_imma");
    ozaki_tc_rows(ctx, oz->tc, S, kp, nr, m, oz->As.get(), false, oz->sA.get(), oz->Bs.get(), true, oz->sB.get(),
                  C + r0 * ldc, ldc, tri);
  }
}

void ozaki_gemm_rows(stgp_ctx* ctx, long long n, int m, int k, const double* A, int lda, const double* B, int ldb,
                     double* C, int ldc) {
  rows_product(ctx, slices_for("STGP_OZAKI_S_ROWS", 6), n, m, k, A, lda, B, ldb, C, ldc);
}

// 32 x 32 tiles through shared memory (the M x M triangular factor, once per product)
__global__ void transpose_kernel(int n, const double* __restrict__ T, int ldt, double* __restrict__ out) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = bx + threadIdx.x, j = by + r;
    t[r][threadIdx.x] = (i < n && j < n) ? T[static_cast<size_t>(j) * ldt + i] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int i = by + threadIdx.x, j = bx + r;
    if (i < n && j < n) out[static_cast<size_t>(j) * n + i] = t[threadIdx.x][r];
  }
}

bool ozaki_trmm_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("STGP_OZAKI_TRMM");  // A/B switch: 0 = the DMMA TRMM
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

void ozaki_trmm_left(stgp_ctx* ctx, const double* T, int ldt, int n, const double* B, int ldb, long long ncols,
                     bool transpose, double* C, int ldc, bool skip) {
  // C(:, r) = op(T) B(:, r): row r of the rows form is column r of B, the B operand's row j is row j
  // of op(T) -- column j of T (transpose) or row j of T, transposed once into scratch
  OzakiState* oz = state(ctx);
  const double* rowsT = T;
  int ldr = ldt;
  if (!transpose) {
    oz->Tt.ensure(static_cast<size_t>(n) * n);
    transpose_kernel<<<dim3((n + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, ctx->stream>>>(n, T, ldt, oz->Tt.get());
    launched(ctx);
    rowsT = oz->Tt.get();
    ldr = n;
  }
  // rows of T^T (columns of T) vanish before the diagonal, rows of T beyond it
  rows_product(ctx, slices_for("STGP_OZAKI_S_TRMM", 7), ncols, n, n, B, ldb, rowsT, ldr, C, ldc,
               skip ? (transpose ? 2 : 1) : 0);
}

// Column-form product C[j ldc + i] = sum_r (fA_r A[j + r lda]) (fB_r B[i + r ldb]) with optional
// per-column factors fA, fB (device vectors).  same: A == B with fA == fB (one slicing pass; the
// tcgen05 kernel loads every slice by its coordinate, so X and Y read the same digits).  keep: the
// digits of A go to the context's kept buffer (tag); kept: A's digits are taken from there instead of
// slicing A.
static void cols_product(stgp_ctx* ctx, int m, long long n, const double* A, int lda, const double* fA, const double* B,
                         int ldb, const double* fB, bool same, uint64_t keep_tag, bool use_kept, double* C, int ldc,
                         bool symmetric = false) {
  const int S = slices_for("STGP_OZAKI_S_COLS", 7);
  OzakiState* oz = state(ctx);
  cudaStream_t st = ctx->stream;
  // chunk of the reduction: exact int32 for the longest diagonal, (S) L 127^2 < 2^31
  const long long lmax = ((1LL << 31) - 1) / (static_cast<long long>(S) * 127 * 127);
  const int L = static_cast<int>(std::min<long long>(lmax / kSlCols * kSlCols, (n + kSlCols - 1) / kSlCols * kSlCols));
  const int nch = static_cast<int>((n + L - 1) / L);
  const long long ldk = static_cast<long long>(S) * L;
  const long long bstride = static_cast<long long>(m) * ldk;
  const size_t sl = static_cast<size_t>(nch) * bstride;
  int8_t* Aslices;
  double* sA;
  if (keep_tag != 0 || use_kept) {
    oz->keep.ensure(sl);
    oz->keep_s.ensure(static_cast<size_t>(nch) * m);
    Aslices = oz->keep.get();
    sA = oz->keep_s.get();
  } else {
    oz->As.ensure(sl);
    oz->sA.ensure(static_cast<size_t>(nch) * m);
    Aslices = oz->As.get();
    sA = oz->sA.get();
  }
  if (!same) {
    oz->Bs.ensure(sl);
    oz->sB.ensure(static_cast<size_t>(nch) * m);
  }
  const dim3 grid(static_cast<unsigned>((n + kSlCols - 1) / kSlCols), (m + 31) / 32);
  // the slicer covers every chunk to its full length L: the padding columns [n, nch L) of the
  // last chunk enter the int8 products and must be zero digits (reused buffers hold old data)
  const int H = slice_halves();
  const int jf = slice_jfast();
  const unsigned nrb = static_cast<unsigned>(static_cast<long long>(nch) * L / (128 * H)), njb = (m + 31) / 32;
  const dim3 sgrid(jf ? njb : nrb, jf ? nrb : njb);
  oz->maxbits.ensure(static_cast<size_t>(nch) * m);
  auto slice = [&](const double* X, int ldx, const double* f, int8_t* fwd, int8_t* rev, double* sc) {
    STGP_CUDA(cudaMemsetAsync(oz->maxbits.get(), 0, sizeof(unsigned long long) * nch * m, st));
    if (colmax_rows())
      colmax_rows_kernel<<<static_cast<unsigned>((n + kMaxRowsPerBlock - 1) / kMaxRowsPerBlock), 256, 0, st>>>(
          m, n, L, X, ldx, f, oz->maxbits.get());
    else
      colmax_kernel<<<grid, 256, 0, st>>>(m, n, L, X, ldx, f, oz->maxbits.get());
    launched(ctx);
    STGP_OZ_SWITCH(S, ({
                     if (H == 1) {
                       const int smem = kS * 32 * sl_row<1>() + 128 * 32 * 8;
                       STGP_CUDA(cudaFuncSetAttribute(slice_cols_kernel<kS, 1>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                       slice_cols_kernel<kS, 1><<<sgrid, 256, smem, st>>>(m, n, L, X, ldx, f, oz->maxbits.get(), fwd,
                                                                          rev, sc, jf);
                     } else {
                       const int smem = kS * 32 * sl_row<2>() + 256 * 32 * 8;
                       STGP_CUDA(cudaFuncSetAttribute(slice_cols_kernel<kS, 2>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                       slice_cols_kernel<kS, 2><<<sgrid, 256, smem, st>>>(m, n, L, X, ldx, f, oz->maxbits.get(), fwd,
                                                                          rev, sc, jf);
                     }
                   }));
    launched(ctx);
  };
  if (!use_kept) slice(A, lda, fA, Aslices, nullptr, sA);
  if (!same) slice(B, ldb, fB, oz->Bs.get(), nullptr, oz->sB.get());
  if (keep_tag != 0) {
    oz->keep_tag = keep_tag;
    oz->keep_m = m;
    oz->keep_n = n;
  }
  const double* sB = same ? sA : oz->sB.get();
  ProfRegion pr(ctx, "oz_imma");
  ozaki_tc_cols(ctx, oz->tc, S, L, nch, m, Aslices, false, sA, same ? Aslices : oz->Bs.get(), false, sB,
                same || symmetric, C, ldc);
}

// per-column factor vector 1 / sqrt(D) (inverse) or sqrt(D)
static const double* col_factors(stgp_ctx* ctx, DevBuf<double>& buf, const double* D, long long n, bool inverse) {
  buf.ensure(static_cast<size_t>(n));
  if (inverse) rsqrt_vec_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(n, D, buf.get());
  else sqrt_vec_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(n, D, buf.get());
  launched(ctx);
  return buf.get();
}

void ozaki_gemm_cols(stgp_ctx* ctx, int m, long long n, const double* A, int lda, const double* B, int ldb, double* C,
                     int ldc, const double* colD) {
  if (m <= 0) return;
  const double* f = colD ? col_factors(ctx, state(ctx)->colf, colD, n, true) : nullptr;
  cols_product(ctx, m, n, A, lda, f, B, ldb, f, A == B && lda == ldb, 0, false, C, ldc);
}

void ozaki_syrk_keep(stgp_ctx* ctx, int m, long long n, const double* A, int lda, const double* D, double* C, int ldc,
                     uint64_t tag) {
  if (m <= 0) return;
  const double* f = col_factors(ctx, state(ctx)->colf, D, n, true);
  cols_product(ctx, m, n, A, lda, f, A, lda, f, true, tag, false, C, ldc);
}

__global__ void sqrt_mul_vec_kernel(long long n, const double* __restrict__ d, const double* __restrict__ g,
                                    double* __restrict__ f) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    f[i] = sqrt(d[i]) * g[i];
}

bool ozaki_gemm_kept(stgp_ctx* ctx, int m, long long n, const double* B, int ldb, const double* D, double* C, int ldc,
                     uint64_t tag, bool symmetric, const double* colmul) {
  OzakiState* oz = state(ctx);
  if (m <= 0 || tag == 0 || oz->keep_tag != tag || oz->keep_m != m || oz->keep_n != n) return false;
  const double* f;
  if (colmul) {
    oz->colf2.ensure(static_cast<size_t>(n));
    sqrt_mul_vec_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(n, D, colmul, oz->colf2.get());
    launched(ctx);
    f = oz->colf2.get();
  } else {
    f = col_factors(ctx, oz->colf2, D, n, false);
  }
  cols_product(ctx, m, n, nullptr, 0, nullptr, B, ldb, f, false, 0, true, C, ldc, symmetric);
  return true;
}

}  // namespace stgp

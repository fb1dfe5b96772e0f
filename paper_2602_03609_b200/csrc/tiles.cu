// Tile-staged column gathers of the VIF algebra (approximations.cpp:277-312, 573-744).
//
// Three steps of a VIF evaluation read, for every row i, the m_v + 1 closure columns of an
// ldm x n column-major matrix (7.3 KB each at M = 906):
//   V'_i   = W_i - sum_a A_ia W_{N_a}                       (build, vprime)
//   Ga_i,s = W_{cl_s} . X_i                                 (gradient rows, SDDMM)
//   Z_i    = sum_a Rv_ia W_{N_a}  -> E_i, F_i                (gradient, ef)
// A row gather re-reads each column once per referencing row (~31x): 249 GB of L2 traffic per
// pass at cfg4.  Here outputs are grouped into tiles of <= 32 space-time neighbours (same time,
// Morton order) whose closures overlap: the union of a tile's source columns (~220 for 32 rows at
// cfg4, scripts/union_probe.py) is staged once per M-chunk into shared memory by cp.async and
// every output of the tile reads its sources from there.  Per-output arithmetic keeps the order
// of the row kernels (same fma chain over a, then the self term), so V' and E/F are bit-identical
// to the row gathers; Ga is a fixed-order sum (deterministic).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "lowrank_common.cuh"
#include "tiles.cuh"

namespace stgp {

namespace {


__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Stage rows [m0, m0 + CH) of the nU union columns of src (ldm x n) into dst[u * CH + c];
// colofs[u] = element offset of union column u (ucol[u] * ldm).
template <int CH>
__device__ __forceinline__ void stage_cols(double* dst, const double* __restrict__ src, const long long* colofs,
                                           int nU, int m0) {
  constexpr unsigned V = CH / 2;  // 16-byte pieces per column chunk
  const unsigned v = threadIdx.x % V;
  const double* s0 = src + m0 + 2 * v;
  double* d0 = dst + 2 * v;
  for (unsigned u = threadIdx.x / V; u < static_cast<unsigned>(nU); u += blockDim.x / V)
    cp_async16(d0 + u * CH, s0 + colofs[u]);
}

struct RowTileArgs {
  int ntiles, m_v, ldm, nch, gchunks;
  const int32_t *tptr, *out, *uptr, *ucol;
  const uint16_t* slot;  // per output position: m_v + 1 union slots (last = self), 0xffff = none
  unsigned long long* next;
};

// Block shape of the row-tile kernels: one output per half-warp (32 outputs = one tile), lane in
// half = row of the M-chunk, so every shared load of a staged column is a 128-byte segment.  A
// thread's coefficients and slot offsets live in registers for the whole item.  Chunks stream
// through a kStages-deep cp.async ring (one barrier per chunk).
constexpr int kCH = 16;
constexpr int kTileBlock = kTileRows * 16;
constexpr int kStages = 4;

struct Ring {
  double* base;
  int stride;  // doubles per stage
  __device__ double* operator[](int b) const { return base + static_cast<size_t>(b) * stride; }
};

// shared double at a byte offset from base
__device__ __forceinline__ double lds_at(const double* base, int byte_off) {
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(base) + byte_off);
}

// Claim the next item; returns -1 when done.
__device__ __forceinline__ int claim(unsigned long long* next, long long items, int* sItem) {
  __syncthreads();
  if (threadIdx.x == 0) *sItem = static_cast<int>(atomicAdd(next, 1ull));
  __syncthreads();
  const int it = *sItem;
  return it < items ? it : -1;
}

// Per-thread slots of output o (half-warp) into registers: byte offset of neighbour a's staged
// element (the zero row `zrow` when absent, with coefficient 0, so the unrolled chains carry no
// predicates: fma(0, 0, acc) = acc), coef[a] = f(a); self_off for the row itself.
template <class F>
__device__ __forceinline__ void load_row_meta(const RowTileArgs& t, int pos, int zrow, int c, int* off, double* coef,
                                              F f, int& self_off) {
  const uint16_t* sl = t.slot + static_cast<size_t>(pos) * (t.m_v + 1);
#pragma unroll
  for (int a = 0; a < 31; ++a) {
    const uint16_t v = a < t.m_v ? __ldg(&sl[a]) : static_cast<uint16_t>(0xffff);
    STGP_DCHECK(v == 0xffff || v < zrow);
    off[a] = static_cast<int>(sizeof(double)) * ((v == 0xffff ? zrow : v) * kCH + c);
    coef[a] = v == 0xffff ? 0.0 : f(a);
  }
  STGP_DCHECK(__ldg(&sl[t.m_v]) < zrow);
  self_off = static_cast<int>(sizeof(double)) * (__ldg(&sl[t.m_v]) * kCH + c);
}

// V' = W B^T over row tiles: V'_i = (sum_a -A_ia W_{N_a}) + W_i, the fma chain of
// lowrank.cu vprime_kernel.  Items = (chunk group, tile), group-major.
__global__ void __launch_bounds__(kTileBlock, 1) tile_vprime_kernel(RowTileArgs t, int ucap, const double* __restrict__ W,
                                                                     const double* __restrict__ A, double* Vp) {
  extern __shared__ double smem[];
  const Ring ring{smem, (ucap + 1) * kCH};
  long long* sU = reinterpret_cast<long long*>(smem + static_cast<size_t>(kStages) * ring.stride);
  __shared__ int sItem;
  const int o = threadIdx.x >> 4, c = threadIdx.x & 15;
  for (int b = 0; b < kStages; ++b)
    if (threadIdx.x < kCH) ring[b][ucap * kCH + threadIdx.x] = 0.0;
  const int ngrp = (t.nch + t.gchunks - 1) / t.gchunks;
  const long long items = static_cast<long long>(ngrp) * t.ntiles;
  for (int item; (item = claim(t.next, items, &sItem)) >= 0;) {
    const int g = item / t.ntiles, tt = item - g * t.ntiles;
    const int o0 = __ldg(&t.tptr[tt]), nout = __ldg(&t.tptr[tt + 1]) - o0;
    const int u0 = __ldg(&t.uptr[tt]), nU = __ldg(&t.uptr[tt + 1]) - u0;
    STGP_DCHECK(nU <= ucap && __ldg(&t.tptr[tt + 1]) - __ldg(&t.tptr[tt]) <= kTileRows);
    for (int e = threadIdx.x; e < nU; e += blockDim.x) sU[e] = static_cast<long long>(__ldg(&t.ucol[u0 + e])) * t.ldm;
    const bool live = o < nout;
    int off[31], self_off = 0;
    double coef[31];
    int row = 0;
    if (live) {
      row = __ldg(&t.out[o0 + o]);
      const double* Ar = A + static_cast<size_t>(row) * t.m_v;
      load_row_meta(t, o0 + o, ucap, c, off, coef, [&](int a) { return -__ldg(&Ar[a]); }, self_off);
    }
    __syncthreads();
    const int q0 = g * t.gchunks, q1 = min(t.nch, q0 + t.gchunks);
#pragma unroll
    for (int b = 0; b < kStages - 1; ++b) {
      if (q0 + b < q1) stage_cols<kCH>(ring[b], W, sU, nU, (q0 + b) * kCH);
      cp_commit();
    }
    for (int q = q0; q < q1; ++q) {
      cp_wait<kStages - 2>();
      __syncthreads();
      {
        const int qn = q + kStages - 1;
        if (qn < q1) stage_cols<kCH>(ring[(qn - q0) % kStages], W, sU, nU, qn * kCH);
        cp_commit();
      }
      if (live) {
        const double* cur = ring[(q - q0) % kStages];
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < 31; ++a) acc += coef[a] * lds_at(cur, off[a]);
        acc += lds_at(cur, self_off);
        Vp[static_cast<size_t>(row) * t.ldm + q * kCH + c] = acc;
      }
    }
    cp_wait<0>();
  }
}

// E_r = X_r / D_r - 2 c0_r V'_r + Z_r - yhat (Bz)_r / D_r,  F_r = c0_r V'_r - Z_r,
// Z_r = sum_a Rv_r[a] W_{N_a}  (lowrank.cu ef_kernel, same arithmetic), over row tiles.  The
// tile's own V' and X chunks are staged with the union.
__global__ void __launch_bounds__(kTileBlock, 1) tile_ef_kernel(RowTileArgs t, int ucap, const double* __restrict__ W,
                                                                 const double* __restrict__ Rv, const double* __restrict__ c0,
                                                                 const double* __restrict__ D, const double* __restrict__ Vp,
                                                                 const double* __restrict__ yhat, const double* __restrict__ Bz,
                                                                 double* X_E, double* F) {
  extern __shared__ double smem[];
  const Ring ring{smem, (ucap + 1 + 2 * kTileRows) * kCH};  // union rows, zero row, V' rows, X rows
  long long* sU = reinterpret_cast<long long*>(smem + static_cast<size_t>(kStages) * ring.stride);
  int* sO = reinterpret_cast<int*>(sU + ucap);
  __shared__ int sItem;
  const int o = threadIdx.x >> 4, c = threadIdx.x & 15;
  for (int b = 0; b < kStages; ++b)
    if (threadIdx.x < kCH) ring[b][ucap * kCH + threadIdx.x] = 0.0;
  const int ngrp = (t.nch + t.gchunks - 1) / t.gchunks;
  const long long items = static_cast<long long>(ngrp) * t.ntiles;
  const int vrow = (ucap + 1) * kCH, xrow = vrow + kTileRows * kCH;
  for (int item; (item = claim(t.next, items, &sItem)) >= 0;) {
    const int g = item / t.ntiles, tt = item - g * t.ntiles;
    const int o0 = __ldg(&t.tptr[tt]), nout = __ldg(&t.tptr[tt + 1]) - o0;
    const int u0 = __ldg(&t.uptr[tt]), nU = __ldg(&t.uptr[tt + 1]) - u0;
    STGP_DCHECK(nU <= ucap && __ldg(&t.tptr[tt + 1]) - __ldg(&t.tptr[tt]) <= kTileRows);
    for (int e = threadIdx.x; e < nU; e += blockDim.x) sU[e] = static_cast<long long>(__ldg(&t.ucol[u0 + e])) * t.ldm;
    if (threadIdx.x < nout) sO[threadIdx.x] = __ldg(&t.out[o0 + threadIdx.x]);
    const bool live = o < nout;
    int off[31], self_off = 0;
    double coef[31];
    int row = 0;
    double cr = 0.0, inv = 0.0, qr = 0.0;
    if (live) {
      row = __ldg(&t.out[o0 + o]);
      const double* Rr = Rv + static_cast<size_t>(row) * t.m_v;
      load_row_meta(t, o0 + o, ucap, c, off, coef, [&](int a) { return __ldg(&Rr[a]); }, self_off);
      inv = 1.0 / __ldg(&D[row]);
      cr = __ldg(&c0[row]);
      qr = __ldg(&Bz[row]) * inv;
    }
    __syncthreads();
    auto stage = [&](int q, double* buf) {
      stage_cols<kCH>(buf, W, sU, nU, q * kCH);
      for (int e = threadIdx.x; e < nout * (kCH / 2); e += blockDim.x) {
        const int oo = e / (kCH / 2), v = e - oo * (kCH / 2);
        const size_t src = static_cast<size_t>(sO[oo]) * t.ldm + q * kCH + 2 * v;
        cp_async16(buf + vrow + oo * kCH + 2 * v, Vp + src);
        cp_async16(buf + xrow + oo * kCH + 2 * v, X_E + src);
      }
    };
    const int q0 = g * t.gchunks, q1 = min(t.nch, q0 + t.gchunks);
#pragma unroll
    for (int b = 0; b < kStages - 1; ++b) {
      if (q0 + b < q1) stage(q0 + b, ring[b]);
      cp_commit();
    }
    for (int q = q0; q < q1; ++q) {
      cp_wait<kStages - 2>();
      __syncthreads();
      {
        const int qn = q + kStages - 1;
        if (qn < q1) stage(qn, ring[(qn - q0) % kStages]);
        cp_commit();
      }
      if (live) {
        const double* cur = ring[(q - q0) % kStages];
        double zr = 0.0;
#pragma unroll
        for (int a = 0; a < 31; ++a) zr = fma(coef[a], lds_at(cur, off[a]), zr);
        const int j = q * kCH + c;
        const size_t gofs = static_cast<size_t>(row) * t.ldm + j;
        const double v = cur[vrow + o * kCH + c], xe = cur[xrow + o * kCH + c];
        X_E[gofs] = xe * inv - 2.0 * cr * v + zr - __ldg(&yhat[j]) * qr;
        F[gofs] = cr * v - zr;
      }
    }
    cp_wait<0>();
  }
}

// Ga(i, s) = W_{cl_s} . X_i for the closure slots s (neighbours 0..m_v-1, self at 31) over row
// tiles: the union columns and the tile's X columns are staged per chunk; half-warp o owns the 32
// (output o, slot) pairs, lane in half = row of the chunk.  Chunk partials stay in registers; one
// 16-lane reduction per pair at the end (fixed order).
__global__ void __launch_bounds__(kTileBlock, 1) tile_ga_kernel(RowTileArgs t, int ucap, const double* __restrict__ W,
                                                                 const double* __restrict__ X, double* Ga) {
  extern __shared__ double smem[];
  const Ring ring{smem, (ucap + 1 + kTileRows) * kCH};  // union rows, zero row, X rows
  long long* sU = reinterpret_cast<long long*>(smem + static_cast<size_t>(kStages) * ring.stride);
  int* sO = reinterpret_cast<int*>(sU + ucap);
  __shared__ int sItem;
  const int o = threadIdx.x >> 4, c = threadIdx.x & 15;
  for (int b = 0; b < kStages; ++b)
    if (threadIdx.x < kCH) ring[b][ucap * kCH + threadIdx.x] = 0.0;
  const int xrow = (ucap + 1) * kCH;
  for (int tt; (tt = claim(t.next, t.ntiles, &sItem)) >= 0;) {
    const int o0 = __ldg(&t.tptr[tt]), nout = __ldg(&t.tptr[tt + 1]) - o0;
    const int u0 = __ldg(&t.uptr[tt]), nU = __ldg(&t.uptr[tt + 1]) - u0;
    STGP_DCHECK(nU <= ucap && __ldg(&t.tptr[tt + 1]) - __ldg(&t.tptr[tt]) <= kTileRows);
    for (int e = threadIdx.x; e < nU; e += blockDim.x) sU[e] = static_cast<long long>(__ldg(&t.ucol[u0 + e])) * t.ldm;
    if (threadIdx.x < nout) sO[threadIdx.x] = __ldg(&t.out[o0 + threadIdx.x]);
    const bool live = o < nout;
    int off[32];
#pragma unroll
    for (int s = 0; s < 32; ++s) off[s] = static_cast<int>(sizeof(double)) * (ucap * kCH + c);
    if (live) {
      const uint16_t* sl = t.slot + static_cast<size_t>(o0 + o) * (t.m_v + 1);
#pragma unroll
      for (int s = 0; s < 31; ++s) {
        const uint16_t v = s < t.m_v ? __ldg(&sl[s]) : static_cast<uint16_t>(0xffff);
        STGP_DCHECK(v == 0xffff || v < ucap);
        off[s] = static_cast<int>(sizeof(double)) * ((v == 0xffff ? ucap : v) * kCH + c);
      }
      off[31] = static_cast<int>(sizeof(double)) * (__ldg(&sl[t.m_v]) * kCH + c);
    }
    __syncthreads();
    auto stage = [&](int q, double* buf) {
      stage_cols<kCH>(buf, W, sU, nU, q * kCH);
      for (int e = threadIdx.x; e < nout * (kCH / 2); e += blockDim.x) {
        const int oo = e / (kCH / 2), v = e - oo * (kCH / 2);
        cp_async16(buf + xrow + oo * kCH + 2 * v, X + static_cast<size_t>(sO[oo]) * t.ldm + q * kCH + 2 * v);
      }
    };
    double acc[32];
#pragma unroll
    for (int s = 0; s < 32; ++s) acc[s] = 0.0;
#pragma unroll
    for (int b = 0; b < kStages - 1; ++b) {
      if (b < t.nch) stage(b, ring[b]);
      cp_commit();
    }
    for (int q = 0; q < t.nch; ++q) {
      cp_wait<kStages - 2>();
      __syncthreads();
      {
        const int qn = q + kStages - 1;
        if (qn < t.nch) stage(qn, ring[qn % kStages]);
        cp_commit();
      }
      if (live) {
        const double* cw = ring[q % kStages];
        const double xv = cw[xrow + o * kCH + c];
#pragma unroll
        for (int s = 0; s < 32; ++s) acc[s] = fma(lds_at(cw, off[s]), xv, acc[s]);
      }
    }
    cp_wait<0>();
#pragma unroll
    for (int s = 0; s < 32; ++s) {
      double v = acc[s];
#pragma unroll
      for (int sh = 8; sh > 0; sh >>= 1) v += __shfl_xor_sync(0xffffffffu, v, sh, 16);
      acc[s] = v;
    }
    if (live) {
      double v0 = 0.0, v1 = 0.0;  // lane c writes slots c and c + 16 (static register indexing)
#pragma unroll
      for (int s = 0; s < 16; ++s)
        if (c == s) {
          v0 = acc[s];
          v1 = acc[s + 16];
        }
      double* dst = Ga + static_cast<size_t>(sO[o]) * 32;
      dst[c] = v0;
      dst[c + 16] = v1;
    }
  }
}

size_t vprime_smem(int ucap) {
  return sizeof(double) * kStages * static_cast<size_t>(ucap + 1) * kCH + sizeof(long long) * ucap;
}
size_t ef_smem(int ucap) {
  return sizeof(double) * kStages * static_cast<size_t>(ucap + 1 + 2 * kTileRows) * kCH + sizeof(long long) * ucap +
         sizeof(int) * kTileRows;
}
size_t ga_smem(int ucap) {
  return sizeof(double) * kStages * static_cast<size_t>(ucap + 1 + kTileRows) * kCH + sizeof(long long) * ucap +
         sizeof(int) * kTileRows;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

template <typename K>
int resident_grid(stgp_ctx* ctx, K kern, size_t smem, long long items, int threads) {
  // the attribute is per function and process-wide: always the device maximum, so that concurrent
  // contexts (in-process ranks) launching with different tile unions never race on it
  static const int max_optin = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v > 0 ? v : 227 * 1024;
  }();
  cudaFuncAttributes fa{};
  STGP_CUDA(cudaFuncGetAttributes(&fa, kern));
  const int dyn_max = max_optin - static_cast<int>(fa.sharedSizeBytes);
  if (static_cast<long long>(smem) > dyn_max) return 0;
  STGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
  int per_sm = 0;
  STGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  return static_cast<int>(std::max<long long>(1, std::min<long long>(items, std::max(1, per_sm) * ctx->num_sms)));
}

// Greedy tiles over outputs in locality order: at most kTileRows outputs and at most ucap distinct
// sources per tile.  srcs(o, f) calls f(source or -1) for each entry of output o.  Returns false
// when one output alone needs more than ucap sources.
template <class Srcs>
bool make_tiles(const std::vector<int32_t>& outs, int n, int ucap, Srcs srcs, std::vector<int32_t>& tptr,
                std::vector<int32_t>& uptr, std::vector<int32_t>& ucol, int& maxU) {
  tptr.assign(1, 0);
  uptr.assign(1, 0);
  ucol.clear();
  std::vector<int32_t> stamp(static_cast<size_t>(n), -1);  // tile that holds column c
  std::vector<int32_t> probe(static_cast<size_t>(n), -1);  // output that last counted c as fresh
  int tile = 0, nout = 0, nU = 0;
  maxU = 0;
  std::vector<int32_t> fresh;
  auto collect = [&](int k) {
    fresh.clear();
    srcs(outs[k], [&](int c) {
      if (c >= 0 && stamp[static_cast<size_t>(c)] != tile && probe[static_cast<size_t>(c)] != k) {
        probe[static_cast<size_t>(c)] = k;
        fresh.push_back(c);
      }
    });
  };
  for (int k = 0; k < static_cast<int>(outs.size()); ++k) {
    collect(k);
    if (static_cast<int>(fresh.size()) > ucap) return false;
    if (nout == kTileRows || nU + static_cast<int>(fresh.size()) > ucap) {
      tptr.push_back(k);
      uptr.push_back(static_cast<int32_t>(ucol.size()));
      maxU = std::max(maxU, nU);
      ++tile;
      nout = nU = 0;
      for (int c : fresh) probe[static_cast<size_t>(c)] = -1;
      collect(k);
    }
    for (int c : fresh) {
      stamp[static_cast<size_t>(c)] = tile;
      ucol.push_back(c);
      ++nU;
    }
    ++nout;
  }
  if (nout > 0) {
    tptr.push_back(static_cast<int32_t>(outs.size()));
    uptr.push_back(static_cast<int32_t>(ucol.size()));
    maxU = std::max(maxU, nU);
  }
  return true;
}

// (time id, Morton code of (x, y)) order of [lo, hi)
std::vector<int32_t> tile_order(const stgp_dataset* ds, int lo, int hi) {
  std::vector<int32_t> out;
  if (hi <= lo) return out;
  double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
  for (int i = lo; i < hi; ++i) {
    x0 = std::min(x0, ds->hx[i]);
    x1 = std::max(x1, ds->hx[i]);
    y0 = std::min(y0, ds->hy[i]);
    y1 = std::max(y1, ds->hy[i]);
  }
  const double sx = x1 > x0 ? 65535.0 / (x1 - x0) : 0.0, sy = y1 > y0 ? 65535.0 / (y1 - y0) : 0.0;
  auto spread = [](uint64_t v) {
    v &= 0xffff;
    v = (v | (v << 8)) & 0x00ff00ff;
    v = (v | (v << 4)) & 0x0f0f0f0f;
    v = (v | (v << 2)) & 0x33333333;
    v = (v | (v << 1)) & 0x55555555;
    return v;
  };
  std::vector<std::pair<uint64_t, int32_t>> key(static_cast<size_t>(hi - lo));
  for (int i = lo; i < hi; ++i) {
    const uint64_t qx = static_cast<uint64_t>((ds->hx[i] - x0) * sx), qy = static_cast<uint64_t>((ds->hy[i] - y0) * sy);
    const uint64_t tk = static_cast<uint64_t>(ds->htid[static_cast<size_t>(i)]);
    key[static_cast<size_t>(i - lo)] = {(tk << 32) | spread(qx) | (spread(qy) << 1), i};
  }
  std::sort(key.begin(), key.end());
  out.resize(key.size());
  for (size_t k = 0; k < key.size(); ++k) out[k] = key[k].second;
  return out;
}

}  // namespace

bool tiles_enabled() {
  static const bool on = env_int("STGP_TILES", 1) != 0;  // A/B switch: 0 = per-row gathers
  return on;
}

// Row tiles over [row_begin, row_end), built once per structure (neighbour sets are fixed).
void ensure_tiles(stgp_structure* s) {
  if (s->tiles_built) return;
  s->tiles_built = true;
  stgp_ctx* ctx = s->ds->ctx;
  cudaStream_t st = ctx->stream;
  const int n = s->n, m_v = s->m_v, rb = s->row_begin, re = s->row_end;
  TileSets& T = s->tiles;
  T.rows.valid = false;
  if (m_v + 1 > 32 || re <= rb) return;
  std::vector<int32_t> nbr(static_cast<size_t>(n) * m_v);
  s->nbr.download(nbr.data(), nbr.size(), st);
  STGP_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> tptr, uptr, ucol;
  // row tiles
  {
    const int ucap = env_int("STGP_TILE_UCAP", 320);
    const std::vector<int32_t> outs = tile_order(s->ds, rb, re);
    auto srcs = [&](int i, auto&& f) {
      for (int a = 0; a < m_v; ++a) f(nbr[static_cast<size_t>(i) * m_v + a]);
      f(i);
    };
    int maxU = 0;
    if (make_tiles(outs, n, ucap, srcs, tptr, uptr, ucol, maxU)) {
      // per output position: union slots of the m_v neighbours and the row itself
      std::vector<uint16_t> slot(outs.size() * static_cast<size_t>(m_v + 1), 0xffff);
      const int nt = static_cast<int>(tptr.size()) - 1;
      std::vector<uint16_t> sl2(static_cast<size_t>(n), 0);  // union slot of a column in the current tile
      for (int t = 0; t < nt; ++t) {
        for (int u = uptr[t]; u < uptr[t + 1]; ++u) sl2[static_cast<size_t>(ucol[u])] = static_cast<uint16_t>(u - uptr[t]);
        for (int k = tptr[t]; k < tptr[t + 1]; ++k) {
          const int i = outs[k];
          for (int a = 0; a <= m_v; ++a) {
            const int c = a < m_v ? nbr[static_cast<size_t>(i) * m_v + a] : i;
            if (c >= 0) slot[static_cast<size_t>(k) * (m_v + 1) + a] = sl2[static_cast<size_t>(c)];
          }
        }
      }
      T.rows.ntiles = nt;
      T.rows.ucap = std::max(maxU, 1);
      T.rows.tptr.upload(tptr.data(), tptr.size(), st);
      T.rows.out.upload(outs.data(), outs.size(), st);
      T.rows.uptr.upload(uptr.data(), uptr.size(), st);
      T.rows.ucol.upload(ucol.data(), ucol.size(), st);
      T.rows.slot.upload(slot.data(), slot.size(), st);
      T.rows.valid = true;
    }
  }
  STGP_CUDA(cudaStreamSynchronize(st));
}

static RowTileArgs row_tile_args(stgp_structure* s, int gchunks) {
  const TileSet& T = s->tiles.rows;
  RowTileArgs t;
  t.ntiles = T.ntiles;
  t.m_v = s->m_v;
  t.ldm = s->lr.ldm;
  t.nch = s->lr.ldm / kCH;
  t.gchunks = gchunks;
  t.tptr = T.tptr.get();
  t.out = T.out.get();
  t.uptr = T.uptr.get();
  t.ucol = T.ucol.get();
  t.slot = T.slot.get();
  t.next = claim_counter(s->ds->ctx);
  return t;
}

// resident grid for a tile kernel, 0 when its shared memory does not fit
template <typename K>
static int tile_grid(stgp_structure* s, K kern, size_t smem, long long items) {
  if (smem > 227 * 1024) return 0;
  return resident_grid(s->ds->ctx, kern, smem, items, kTileBlock);
}

static bool tiles_ready(stgp_structure* s) {
  if (!tiles_enabled() || s->lr.ldm % kCH) return false;
  ensure_tiles(s);
  return s->tiles.rows.valid;
}

static int group_chunks() {
  static const int g = std::max(1, env_int("STGP_TILE_G", 19));  // M-chunks per work item
  return g;
}

bool tile_vprime(stgp_structure* s, const double* W, const double* A, double* Vp) {
  if (!tiles_ready(s)) return false;
  stgp_ctx* ctx = s->ds->ctx;
  RowTileArgs t = row_tile_args(s, group_chunks());
  const int ucap = s->tiles.rows.ucap;
  const size_t sm = vprime_smem(ucap);
  const long long items = static_cast<long long>((t.nch + t.gchunks - 1) / t.gchunks) * t.ntiles;
  const int grid = tile_grid(s, tile_vprime_kernel, sm, items);
  if (grid == 0) return false;
  tile_vprime_kernel<<<grid, kTileBlock, sm, ctx->stream>>>(t, ucap, W, A, Vp);
  launched(ctx);
  return true;
}

bool tile_ef(stgp_structure* s, const double* W, const double* Rv, const double* c0, const double* D,
             const double* Vp, const double* yhat, const double* Bz, double* X_E, double* F) {
  if (!tiles_ready(s)) return false;
  stgp_ctx* ctx = s->ds->ctx;
  RowTileArgs t = row_tile_args(s, group_chunks());
  const int ucap = s->tiles.rows.ucap;
  const size_t sm = ef_smem(ucap);
  const long long items = static_cast<long long>((t.nch + t.gchunks - 1) / t.gchunks) * t.ntiles;
  const int grid = tile_grid(s, tile_ef_kernel, sm, items);
  if (grid == 0) return false;
  tile_ef_kernel<<<grid, kTileBlock, sm, ctx->stream>>>(t, ucap, W, Rv, c0, D, Vp, yhat, Bz, X_E, F);
  launched(ctx);
  return true;
}

bool tile_ga(stgp_structure* s, const double* W, const double* X, double* Ga) {
  if (!tiles_ready(s)) return false;
  stgp_ctx* ctx = s->ds->ctx;
  RowTileArgs t = row_tile_args(s, 1);
  const int ucap = s->tiles.rows.ucap;
  const size_t sm = ga_smem(ucap);
  const int grid = tile_grid(s, tile_ga_kernel, sm, t.ntiles);
  if (grid == 0) return false;
  tile_ga_kernel<<<grid, kTileBlock, sm, ctx->stream>>>(t, ucap, W, X, Ga);
  launched(ctx);
  return true;
}

}  // namespace stgp

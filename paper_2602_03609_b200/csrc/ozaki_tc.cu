// Hand-written sm_100a int8 tensor-core kernel for the Ozaki products (ozaki.cu): TMA-fed tcgen05.mma
// kind::i8 with every digit diagonal accumulated in its own TMEM block and the FP64 recombination in the
// epilogue, so the exact int32 partial products never leave the SM.
//
// Operands are the int8 digit slices the slicers of ozaki.cu write (7-bit digits, per-row power-of-two
// scales).  For an output tile of 128 X rows x 64 Y rows the kernel keeps S accumulators
//     C_d[x][y] = sum_{s + t = d} sum_k X_s[x][k] Y_t[y][k],     d = 2 .. S + 1,
// in TMEM columns (d - 2) * 64 .. (d - 2) * 64 + 63 (S <= 8: at most 512 columns), fed one 32-byte K step
// at a time: each pipeline stage holds the S slices of both operands for that K step (TMA, 32-byte
// swizzle), and the single MMA thread issues the S (S + 1) / 2 pair products of the stage.  The epilogue
// warps read the S accumulators back (tcgen05.ld), sum them from the smallest diagonal up in FP64
// (exact power-of-two weights, one rounding per add, the order of the former combine kernels) and scale
// by the row / column scales:
//   rows form  out[x ldo + y]  = (sum_d 2^-7d C_d) sx[x] sy[y]                        (one chunk)
//   cols form  out[x ldo + y] += (sum_d 2^-7d C_d) (sx[c nx + x] sy[c ny + y])  over reduction chunks c
// (a chunk keeps every diagonal exact in int32).  The cols form splits its chunks over `groups` CTAs per
// tile; group partials are summed in group order by ozaki_tc_reduce (deterministic).
//
// Warp roles (192 threads, one CTA per SM, persistent over the work items):
//   warp 0: TMA producer; warp 1: TMEM owner and MMA issuer; warps 2-5: epilogue (TMEM lane quarter
//   warp % 4).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>

#include "lowrank_common.cuh"
#include "ozaki.cuh"

namespace stgp {
namespace {

constexpr int kBM = 128;     // X rows per tile = TMEM lanes = MMA M
constexpr int kBN = 64;      // Y rows per tile = MMA N = TMEM columns per diagonal
constexpr int kBK = 32;      // int8 K per stage (one MMA K step, one 32-byte swizzle row)
// pipeline depth: as many S * 6 KB stages as fit in 220 KB of shared memory, at most STGP_TC_STAGES_MAX
#ifndef STGP_TC_STAGES_MAX
#define STGP_TC_STAGES_MAX 4
#endif
template <int S, int BN = 64>
constexpr int stages_for() {
  constexpr int fit = (220 * 1024) / (S * (128 * 32 + BN * 32));
  return fit < STGP_TC_STAGES_MAX ? fit : STGP_TC_STAGES_MAX;
}
constexpr int kThreads = 192;
constexpr int kTileX = kBM * kBK;  // bytes of one X slice tile
constexpr int kTileY = kBN * kBK;


struct TcArgs {
  int S;
  int kblocks;            // K steps per chunk
  int nx, ny;             // valid X / Y rows
  int nchunks, groups;    // reduction chunks and the split of a tile's chunks over CTAs
  int x_rev, y_rev;       // slice s (1-based) sits at slice coordinate rev ? S - s : s - 1
  int cols;               // 0: rows form (one chunk, write), 1: cols form (accumulate over chunks)
  int nitems;
  const int4* items;      // (x group, y group, split group, K-step range kb0 | kb1 << 16 or 0 = all)
  const double* sx;       // scales: rows form sx[x]; cols form sx[c nx + x]
  const double* sy;
  double* out;            // out[x ldo + y] (+ group * part_stride in the cols form with groups > 1)
  long long ldo, part_stride;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load4(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// the same, multicast to every CTA of the cluster in mask (data and the mbarrier signal land at the same
// shared-memory offsets in each destination CTA)
__device__ __forceinline__ void tma_load4_mc(const CUtensorMap* map, void* dst, uint64_t* bar, int c0, int c1, int c2,
                                             int c3, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// K-major operand tile of rows x 32 bytes written by TMA with 32-byte swizzling: core matrices of 8 rows
// x 16 bytes, 8-row groups 256 bytes apart (SBO), layout type SWIZZLE_32B, descriptor version 1
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(256 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(6) << 61);
}
// instruction descriptor: kind::i8, signed int8 A and B, int32 D, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(kBM >> 4) << 24);
}
constexpr uint32_t kIdesc = idesc_i8(kBN);
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate,
                                       uint32_t idesc = kIdesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(0u));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// arrive on the barrier at this offset in every CTA of the mask once this thread's MMAs are done
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(mask)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// exact int32 -> double without the quarter-rate I2F.F64: 2^52 + 2^31 + v has v + 2^31 as its low word
__device__ __forceinline__ double i32_to_f64(int v) {
  return __hiloint2double(0x43300000, v ^ static_cast<int>(0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}

__device__ __forceinline__ void chunk_range(const TcArgs& a, int g, int& c0, int& c1) {
  c0 = static_cast<int>(static_cast<long long>(a.nchunks) * g / a.groups);
  c1 = static_cast<int>(static_cast<long long>(a.nchunks) * (g + 1) / a.groups);
}

// Clusters of CX x CY CTAs (rank r = rx CY + ry) compute CX X tiles x CY Y tiles.  The CY CTAs of one
// X tile (same rx) each load 128 / CY of its rows and multicast them to the others; the CX CTAs of one
// Y tile (same ry) each load 64 / CX of its rows likewise.  A stage slot is written by the CTA's X
// group and Y group (CX + CY - 1 CTAs), so each CTA's MMA commit arrives on the empty barrier of every
// CTA of both groups.  Items are cluster items (x group, y group, split group).
// BN: Y rows per tile (64, or 32 with two TMEM accumulator sets so that the epilogue of one item
// overlaps the MMAs of the next: S * 32 * 2 <= 512 columns).
template <int S, int CX, int CY, int BN = kBN>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_tc_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy, TcArgs a) {
  constexpr int CL = CX * CY;
  constexpr int kTY = BN * kBK;                 // bytes of one Y slice tile
  constexpr int NSET = BN == kBN ? 1 : 2;       // TMEM accumulator sets
  constexpr int kTPer = 256 / BN;               // Y slices per MMA (N <= 256)
  static_assert(NSET * S * BN <= 512, "TMEM columns");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned stage buffers: [stage][X slices S x 4 KB | Y slices S x 2 KB]
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kStageBytes = S * (kTileX + kTY);
  constexpr int kStages = stages_for<S, BN>();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = CL > 1 ? static_cast<int>(cluster_rank()) : 0;
  const int rx = rank / CY, ry = rank % CY;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  // multicast masks: the X group (same rx) and the Y group (same ry); their union releases the stages
  uint16_t mask_x = 0, mask_y = 0;
  for (int j = 0; j < CY; ++j) mask_x |= static_cast<uint16_t>(1u << (rx * CY + j));
  for (int i = 0; i < CX; ++i) mask_y |= static_cast<uint16_t>(1u << (i * CY + ry));
  const uint16_t mask_xy = static_cast<uint16_t>(mask_x | mask_y);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CX + CY - 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&tmem_empty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 512 columns (S diagonals x 64)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmy)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // every CTA's barriers initialised before remote arrivals
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = cid; it < a.nitems; it += ncl) {
        const int4 job = a.items[it];
        const int xt = job.x * CX + rx, yt = job.y * CY + ry;
        int c0, c1;
        chunk_range(a, job.z, c0, c1);
        const int kb0 = job.w & 0xffff, kb1 = job.w ? job.w >> 16 : a.kblocks;
        for (int c = c0; c < c1; ++c)
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            unsigned char* st = smem + stage * kStageBytes;
            mbar_expect_tx(&full[stage], kStageBytes);
#pragma unroll
            for (int s = 1; s <= S; ++s) {
              if (CY == 1)
                tma_load4(&tmx, st + (s - 1) * kTileX, &full[stage], kb * kBK, a.x_rev ? S - s : s - 1, xt * kBM, c);
              else
                tma_load4_mc(&tmx, st + (s - 1) * kTileX + ry * (kTileX / CY), &full[stage], kb * kBK,
                             a.x_rev ? S - s : s - 1, xt * kBM + ry * (kBM / CY), c, mask_x);
            }
#pragma unroll
            for (int t = 1; t <= S; ++t) {
              if (CX == 1)
                tma_load4(&tmy, st + S * kTileX + (t - 1) * kTY, &full[stage], kb * kBK, a.y_rev ? S - t : t - 1,
                          yt * BN, c);
              else
                tma_load4_mc(&tmy, st + S * kTileX + (t - 1) * kTY + rx * (kTY / CX), &full[stage], kb * kBK,
                             a.y_rev ? S - t : t - 1, yt * BN + rx * (BN / CX), c, mask_y);
            }
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ----
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, acc_n = 0;  // acc_n: accumulations issued (set = acc_n % NSET)
      for (int it = cid; it < a.nitems; it += ncl) {
        const int4 job = a.items[it];
        int c0, c1;
        chunk_range(a, job.z, c0, c1);
        const int kb0 = job.w & 0xffff, kb1 = job.w ? job.w >> 16 : a.kblocks;
        for (int c = c0; c < c1; ++c, ++acc_n) {
          const int set = NSET == 1 ? 0 : static_cast<int>(acc_n & 1);
          const uint32_t sph = NSET == 1 ? (acc_n & 1) : ((acc_n >> 1) & 1);
          mbar_wait(&tmem_empty[set], sph ^ 1);  // the epilogue has read this set's previous accumulators
          tc_fence_after();
          const uint32_t tset = tmem + static_cast<uint32_t>(set * S * BN);
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sbase = smem_u32(smem + stage * kStageBytes);
            // For X slice s the pairs (s, t), t = 1 .. S + 1 - s, feed the consecutive diagonals s - 1 .. S - 1,
            // and the Y slices t are consecutive 64-row tiles: one MMA with N = 64 (S + 1 - s) (<= 256 per
            // instruction) covers them all -- S (S + 1) / 2 pair products in 2 S - S / 4 instructions.
#pragma unroll
            for (int s = 1; s <= S; ++s) {
              const uint64_t da = smem_desc(sbase + (s - 1) * kTileX);
              const int nt = S + 1 - s;
#pragma unroll
              for (int t0 = 1; t0 <= nt; t0 += kTPer) {
                const int cnt = nt - t0 + 1 < kTPer ? nt - t0 + 1 : kTPer;
                const uint64_t db = smem_desc(sbase + S * kTileX + (t0 - 1) * kTY);
                // diagonals s + t0 - 2 ..; the first product (s = 1) of the chunk's first K step starts them
                STGP_DCHECK(set * S * BN + (s + t0 - 2 + cnt) * BN <= 512);
                mma_i8(tset + (s + t0 - 2) * BN, da, db, (kb > kb0 || s > 1) ? 1u : 0u, idesc_i8(BN * cnt));
              }
            }
            if (CL == 1) mma_commit(&empty[stage]);  // frees the stage once these MMAs have read it
            else mma_commit_mc(&empty[stage], mask_xy);  // in every CTA that writes into this CTA's stages
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit(&tmem_full[set]);
        }
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: warps 2..5, TMEM lanes 32 (warp % 4) .. + 31 ----
    const int quarter = warp & 3;
    const uint32_t lane_addr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    uint32_t acc_n = 0;  // accumulations consumed, as issued
    for (int it = cid; it < a.nitems; it += ncl) {
      const int4 job = a.items[it];
      int c0, c1;
      chunk_range(a, job.z, c0, c1);
      const int x = (job.x * CX + rx) * kBM + quarter * 32 + lane;
      const int y0 = (job.y * CY + ry) * BN;
      if (!a.cols) {
        // rows form (one chunk, written once): per 8 columns the S diagonals are read with one wait,
        // combined, scaled and stored; the accumulators are released as soon as the last read lands.
        // Same operations and order as the column form's combine (bit-identical results).
        const int set = NSET == 1 ? 0 : static_cast<int>(acc_n & 1);
        mbar_wait(&tmem_full[set], NSET == 1 ? (acc_n & 1) : ((acc_n >> 1) & 1));
        ++acc_n;
        tc_fence_after();
        const uint32_t lset = lane_addr + static_cast<uint32_t>(set * S * BN);
        const double sxv = x < a.nx ? a.sx[x] : 0.0;
        double* o = a.out + static_cast<long long>(x) * a.ldo + y0;
        const int ny = min(BN, a.ny - y0);
        const bool vec = ny == BN && (reinterpret_cast<uintptr_t>(o) & 15) == 0;
#pragma unroll
        for (int q = 0; q < BN / 8; ++q) {
          int v[S][8];
#pragma unroll
          for (int d = 0; d < S; ++d) tmem_ld8(lset + d * BN + q * 8, v[d]);
          tmem_wait_ld();
          if (q == BN / 8 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[set]);
          }
          double sq[8];
          double w = 0x1p-14;
#pragma unroll
          for (int d = 0; d < S - 1; ++d) w *= 0x1p-7;  // 2^-7(S+1)
#pragma unroll
          for (int d = S - 1; d >= 0; --d) {
#pragma unroll
            for (int e = 0; e < 8; ++e) sq[e] = d == S - 1 ? i32_to_f64(v[d][e]) * w : fma(i32_to_f64(v[d][e]), w, sq[e]);
            w *= 128.0;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int y = y0 + q * 8 + e;
            sq[e] = sq[e] * sxv * (y < a.ny ? __ldg(&a.sy[y]) : 0.0);
          }
          if (x < a.nx) {
            if (vec) {
#pragma unroll
              for (int e = 0; e < 8; e += 2) *reinterpret_cast<double2*>(o + q * 8 + e) = make_double2(sq[e], sq[e + 1]);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (q * 8 + e < ny) o[q * 8 + e] = sq[e];
            }
          }
        }
        continue;
      }
      double acc[BN];
#pragma unroll
      for (int e = 0; e < BN; ++e) acc[e] = 0.0;
      for (int c = c0; c < c1; ++c) {
        const int set = NSET == 1 ? 0 : static_cast<int>(acc_n & 1);
        mbar_wait(&tmem_full[set], NSET == 1 ? (acc_n & 1) : ((acc_n >> 1) & 1));
        ++acc_n;
        tc_fence_after();
        const uint32_t lset = lane_addr + static_cast<uint32_t>(set * S * BN);
        const double sxv = x < a.nx ? a.sx[static_cast<size_t>(a.cols ? c : 0) * a.nx + x] : 0.0;
#pragma unroll
        for (int q = 0; q < BN / 16; ++q) {
          // smallest diagonal first: exact products by powers of two, one rounding per add
          double sq[16];
          double w = 0x1p-14;
#pragma unroll
          for (int d = 0; d < S - 1; ++d) w *= 0x1p-7;  // 2^-7(S+1)
#pragma unroll
          for (int d = S - 1; d >= 0; --d) {
            int v[16];
            tmem_ld16(lset + d * BN + q * 16, v);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) sq[e] = d == S - 1 ? static_cast<double>(v[e]) * w : fma(static_cast<double>(v[e]), w, sq[e]);
            w *= 128.0;
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int y = y0 + q * 16 + e;
            const double syv = y < a.ny ? __ldg(&a.sy[static_cast<size_t>(a.cols ? c : 0) * a.ny + y]) : 0.0;
            if (a.cols) acc[q * 16 + e] = fma(sq[e], sxv * syv, acc[q * 16 + e]);
            else acc[q * 16 + e] = sq[e] * sxv * syv;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty[set]);
      }
      if (x < a.nx) {
        double* o = a.out + (a.cols && a.groups > 1 ? job.z * a.part_stride : 0) + static_cast<long long>(x) * a.ldo + y0;
        const int ny = min(BN, a.ny - y0);
        if (ny == BN && (reinterpret_cast<uintptr_t>(o) & 15) == 0) {
#pragma unroll
          for (int e = 0; e < BN; e += 2) *reinterpret_cast<double2*>(o + e) = make_double2(acc[e], acc[e + 1]);
        } else {
#pragma unroll
          for (int e = 0; e < BN; ++e)
            if (e < ny) o[e] = acc[e];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// C (m x m, ldc) = sum_g P_g in group order; lower_only: then mirror the strictly upper triangle
__global__ void reduce_groups_kernel(int nx, int ny, int groups, const double* __restrict__ P, long long ldp,
                                     long long pstride, double* __restrict__ C, long long ldc) {
  const long long total = static_cast<long long>(nx) * ny;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long x = e / ny, y = e - x * ny;
    double s = P[x * ldp + y];
    for (int g = 1; g < groups; ++g) s += P[g * pstride + x * ldp + y];
    C[x * ldc + y] = s;
  }
}
// symmetric products: rows x < y were not computed; C[x][y] = C[y][x] (bitwise: the products commute)
__global__ void mirror_upper_kernel(int m, double* __restrict__ C, long long ldc) {
  const long long total = static_cast<long long>(m) * m;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long x = e / m, y = e - x * m;
    if (y > x) C[x * ldc + y] = C[y * ldc + x];
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw Error(kInternal, "ozaki_tc: cuTensorMapEncodeTiled is unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 4-D map over int8 digits: (K bytes, slice, row, chunk) with byte strides (1, slice_stride, row_stride,
// chunk_stride); box (32, 1, box_rows, 1), 32-byte swizzle, out-of-range rows read as zero digits
CUtensorMap make_map(const int8_t* base, long long kext, int S, long long rows, int nch, long long slice_stride,
                     long long row_stride, long long chunk_stride, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(kext), static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(nch)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(slice_stride), static_cast<cuuint64_t>(row_stride),
                                 static_cast<cuuint64_t>(chunk_stride)};
  const cuuint32_t box[4] = {static_cast<cuuint32_t>(kBK), 1u, static_cast<cuuint32_t>(box_rows), 1u};
  const cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(kInternal, "ozaki_tc: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

template <int S, int CX, int CY, int BN = kBN>
void launch_tc(stgp_ctx* ctx, const CUtensorMap& tx, const CUtensorMap& ty, const TcArgs& a) {
  constexpr int CL = CX * CY;
  // at least 116 KB so that one CTA holds an SM: it owns all 512 TMEM columns
  constexpr int smem = std::max(stages_for<S, BN>() * S * (kTileX + BN * kBK) + 1024 + 256, 116 * 1024);
  static int max_clusters = 0;
  if (max_clusters == 0) {
    STGP_CUDA(cudaFuncSetAttribute(ozaki_tc_kernel<S, CX, CY, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    max_clusters = ctx->num_sms / CL;
    if (CL > 1) {
      cudaLaunchConfig_t q{};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.gridDim = dim3(CL * max_clusters);
      q.blockDim = dim3(kThreads);
      q.dynamicSmemBytes = smem;
      q.attrs = at;
      q.numAttrs = 1;
      int mc = 0;
      if (cudaOccupancyMaxActiveClusters(&mc, ozaki_tc_kernel<S, CX, CY, BN>, &q) == cudaSuccess && mc > 0)
        max_clusters = mc;
      (void)cudaGetLastError();
    }
  }
  const int clusters = std::min(a.nitems, max_clusters);
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(clusters * CL);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  STGP_CUDA(cudaLaunchKernelEx(&cfg, ozaki_tc_kernel<S, CX, CY, BN>, tx, ty, a));
  launched(ctx);
}

template <int CX, int CY, int BN = kBN>
void dispatch(stgp_ctx* ctx, int S, const CUtensorMap& tx, const CUtensorMap& ty, const TcArgs& a) {
  switch (S) {
    case 2: launch_tc<2, CX, CY, BN>(ctx, tx, ty, a); break;
    case 3: launch_tc<3, CX, CY, BN>(ctx, tx, ty, a); break;
    case 4: launch_tc<4, CX, CY, BN>(ctx, tx, ty, a); break;
    case 5: launch_tc<5, CX, CY, BN>(ctx, tx, ty, a); break;
    case 6: launch_tc<6, CX, CY, BN>(ctx, tx, ty, a); break;
    case 7: launch_tc<7, CX, CY, BN>(ctx, tx, ty, a); break;
    case 8: launch_tc<8, CX, CY, BN>(ctx, tx, ty, a); break;
    default: throw Error(kConfig, "ozaki_tc: slice count must lie in [2, 8]");
  }
}

// Cluster shape per product form: CY CTAs share (multicast) an X tile, CX CTAs a Y tile.
// STGP_OZAKI_CLUSTER=1|2|4 sets CY and STGP_OZAKI_CLUSTER_X=1|2 sets CX for every form.  Measured at
// cfg4 (A/B, one box): the rows form (X = K^-1 V') and the symmetric column form (K) run best with
// CY = 2 (24.8 -> 23.6 and 23.5 -> 22.9 ms), the general column form (V'F^T) with CY = 4 (30.0 -> 29.0 ms).
enum class TcForm { kRows, kColsSym, kCols };
struct TcCluster {
  int cx, cy;
};
TcCluster cluster_shape(TcForm f) {
  static const int env_y = [] {
    const char* e = std::getenv("STGP_OZAKI_CLUSTER");
    const int v = e ? std::atoi(e) : 0;
    return v == 1 || v == 2 || v == 4 ? v : 0;
  }();
  static const int env_x = [] {
    const char* e = std::getenv("STGP_OZAKI_CLUSTER_X");
    const int v = e ? std::atoi(e) : 0;
    return v == 1 || v == 2 ? v : 0;
  }();
  // per-form overrides (tuning): STGP_OZAKI_CLUSTER_ROWS / _SYM / _COLS set CY for one form
  static const int env_form[3] = {
      [] { const char* e = std::getenv("STGP_OZAKI_CLUSTER_ROWS"); const int v = e ? std::atoi(e) : 0; return v == 1 || v == 2 || v == 4 ? v : 0; }(),
      [] { const char* e = std::getenv("STGP_OZAKI_CLUSTER_SYM"); const int v = e ? std::atoi(e) : 0; return v == 1 || v == 2 || v == 4 ? v : 0; }(),
      [] { const char* e = std::getenv("STGP_OZAKI_CLUSTER_COLS"); const int v = e ? std::atoi(e) : 0; return v == 1 || v == 2 || v == 4 ? v : 0; }()};
  TcCluster c{1, f == TcForm::kCols ? 4 : 2};
  if (env_y) c.cy = env_y;
  if (env_form[static_cast<int>(f)]) c.cy = env_form[static_cast<int>(f)];
  if (env_x) c.cx = env_x;
  if (c.cx * c.cy > 4) c.cy = 4 / c.cx;  // instantiated shapes: 1x1, 1x2, 1x4, 2x1, 2x2
  return c;
}

void run(stgp_ctx* ctx, int S, TcCluster c, const CUtensorMap& tx, const CUtensorMap& ty, const TcArgs& a,
         int bn = kBN) {
  if (bn == 32) {  // rows form with two TMEM sets (1-D clusters only)
    if (c.cy == 4) dispatch<1, 4, 32>(ctx, S, tx, ty, a);
    else if (c.cy == 2) dispatch<1, 2, 32>(ctx, S, tx, ty, a);
    else dispatch<1, 1, 32>(ctx, S, tx, ty, a);
    return;
  }
  if (c.cx == 2) {
    if (c.cy == 2) dispatch<2, 2>(ctx, S, tx, ty, a);
    else dispatch<2, 1>(ctx, S, tx, ty, a);
  } else if (c.cy == 4) {
    dispatch<1, 4>(ctx, S, tx, ty, a);
  } else if (c.cy == 2) {
    dispatch<1, 2>(ctx, S, tx, ty, a);
  } else {
    dispatch<1, 1>(ctx, S, tx, ty, a);
  }
}

}  // namespace

struct OzakiTcState {
  DevBuf<int4> items;
  DevBuf<double> part;
};

void ozaki_tc_release(OzakiTcState* s) { delete s; }

static OzakiTcState* tc_state(OzakiTcState*& s) {
  if (!s) s = new OzakiTcState();
  return s;
}

// rows form: out[x ldo + y] = sx[x] sy[y] sum_d 2^-7d sum_{s+t=d} X_s[x] . Y_t[y]; X digits at
// xd[x ldk + slot(s) kp + k], Y digits likewise (ldk = S kp, kp a multiple of 32).  tri: the Y rows are
// those of a triangular factor -- row y vanishes beyond k = y (1, lower) or before it (2, upper) -- and
// each Y group's K loop stops (starts) at the group's last (first) row: half the int8 work.
void ozaki_tc_rows(stgp_ctx* ctx, OzakiTcState*& st, int S, int kp, long long nx, int ny, const int8_t* xd, bool x_rev,
                   const double* sx, const int8_t* yd, bool y_rev, const double* sy, double* out, long long ldo,
                   int tri) {
  if (kp % kBK) throw Error(kInternal, "ozaki_tc_rows: kp must be a multiple of 32");
  OzakiTcState* s = tc_state(st);
  const long long ldk = static_cast<long long>(S) * kp;
  const TcCluster cs = cluster_shape(TcForm::kRows);
  // Y tiles of 32 rows with two TMEM accumulator sets (STGP_OZAKI_ROWS_BN=32; 1-D clusters) or of 64
  static const int env_bn = [] {
    const char* e = std::getenv("STGP_OZAKI_ROWS_BN");
    return e && std::atoi(e) == 32 ? 32 : kBN;
  }();
  const int bn = cs.cx == 1 ? env_bn : kBN;
  const CUtensorMap tx = make_map(xd, kp, S, nx, 1, kp, ldk, nx * ldk, kBM / cs.cy);
  const CUtensorMap ty = make_map(yd, kp, S, ny, 1, kp, ldk, static_cast<long long>(ny) * ldk, bn / cs.cx);
  const int tiles_x = static_cast<int>((nx + kBM - 1) / kBM), tiles_y = (ny + bn - 1) / bn;
  const int groups_x = (tiles_x + cs.cx - 1) / cs.cx, groups_y = (tiles_y + cs.cy - 1) / cs.cy;
  const int kblocks = kp / kBK;
  std::vector<int> krange(groups_y, 0);
  for (int gy = 0; tri && gy < groups_y; ++gy) {
    const int y0 = gy * cs.cy * bn, y1 = std::min(ny, (gy + 1) * cs.cy * bn);  // rows [y0, y1)
    const int kb0 = tri == 2 ? y0 / kBK : 0;
    const int kb1 = tri == 1 ? std::min(kblocks, (y1 + kBK - 1) / kBK) : kblocks;
    krange[gy] = kb0 | (kb1 << 16);
  }
  std::vector<int4> items;
  items.reserve(static_cast<size_t>(groups_x) * groups_y);
  // Y groups fastest: the clusters in flight share one X block in L2.  With triangle-cut K ranges the
  // items differ in cost; the Y order is rotated by the X group so that the clusters' strided shares
  // (item cid + t * clusters) mix short and long items instead of repeating the same Y groups.
  for (int gx = 0; gx < groups_x; ++gx)
    for (int j = 0; j < groups_y; ++j) {
      const int gy = tri ? (j + gx) % groups_y : j;
      items.push_back(make_int4(gx, gy, 0, krange[gy]));
    }
  s->items.upload(items.data(), items.size(), ctx->stream);
  TcArgs a{};
  a.S = S;
  a.kblocks = kblocks;
  a.nx = static_cast<int>(nx);
  a.ny = ny;
  a.nchunks = 1;
  a.groups = 1;
  a.x_rev = x_rev;
  a.y_rev = y_rev;
  a.cols = 0;
  a.nitems = static_cast<int>(items.size());
  a.items = s->items.get();
  a.sx = sx;
  a.sy = sy;
  a.out = out;
  a.ldo = ldo;
  run(ctx, S, cs, tx, ty, a, bn);
}

// cols form: C[x ldc + y] = sum_c (sx[c m + x] sy[c m + y]) sum_d 2^-7d sum_{s+t=d} X_s,c[x] . Y_t,c[y];
// digits at d[((c m + row) S + slot(s)) L + k]; symmetric: X and Y are one matrix, only tiles reaching
// the lower triangle are computed and the upper triangle is mirrored
void ozaki_tc_cols(stgp_ctx* ctx, OzakiTcState*& st, int S, int L, int nch, int m, const int8_t* xd, bool x_rev,
                   const double* sx, const int8_t* yd, bool y_rev, const double* sy, bool symmetric, double* C,
                   long long ldc) {
  if (L % kBK) throw Error(kInternal, "ozaki_tc_cols: L must be a multiple of 32");
  OzakiTcState* s = tc_state(st);
  const long long rs = static_cast<long long>(S) * L;
  const TcCluster cs = cluster_shape(symmetric ? TcForm::kColsSym : TcForm::kCols);
  const int CL = cs.cx * cs.cy;
  const CUtensorMap tx = make_map(xd, L, S, m, nch, L, rs, static_cast<long long>(m) * rs, kBM / cs.cy);
  const CUtensorMap ty = make_map(yd, L, S, m, nch, L, rs, static_cast<long long>(m) * rs, kBN / cs.cx);
  const int tiles_x = (m + kBM - 1) / kBM, tiles_y = (m + kBN - 1) / kBN;
  const int groups_x = (tiles_x + cs.cx - 1) / cs.cx, groups_y = (tiles_y + cs.cy - 1) / cs.cy;
  std::vector<int2> tiles;  // (x group, y group): kept when one of its tiles reaches the lower triangle
  for (int gx = 0; gx < groups_x; ++gx)
    for (int gy = 0; gy < groups_y; ++gy)
      if (!symmetric || gy * cs.cy * kBN < (gx + 1) * cs.cx * kBM) tiles.push_back(make_int2(gx, gy));
  // split the chunks of each tile over G clusters so the work items fill whole waves of the SMs
  const int nt = static_cast<int>(tiles.size());
  const int slots = std::max(1, ctx->num_sms / CL);
  int G = 1;
  double best = 0.0;
  for (int g = 1; g <= std::min(nch, 16); ++g) {
    const long long it = static_cast<long long>(nt) * g;
    const long long waves = (it + slots - 1) / slots;
    const double eff = static_cast<double>(it) / (waves * slots) * (1.0 - 0.02 * (g - 1));
    if (eff > best + 1e-9) {
      best = eff;
      G = g;
    }
  }
  std::vector<int4> items;
  for (int g = 0; g < G; ++g)
    for (const int2& t : tiles) items.push_back(make_int4(t.x, t.y, g, 0));
  s->items.upload(items.data(), items.size(), ctx->stream);
  TcArgs a{};
  a.S = S;
  a.kblocks = L / kBK;
  a.nx = m;
  a.ny = m;
  a.nchunks = nch;
  a.groups = G;
  a.x_rev = x_rev;
  a.y_rev = y_rev;
  a.cols = 1;
  a.nitems = static_cast<int>(items.size());
  a.items = s->items.get();
  a.sx = sx;
  a.sy = sy;
  const long long ldp = (m + 1) / 2 * 2;
  if (G > 1) {
    a.part_stride = static_cast<long long>(m) * ldp;
    s->part.ensure(static_cast<size_t>(G) * a.part_stride);
    a.out = s->part.get();
    a.ldo = ldp;
  } else {
    a.out = C;
    a.ldo = ldc;
  }
  run(ctx, S, cs, tx, ty, a);
  if (G > 1) {
    reduce_groups_kernel<<<grid_for(static_cast<long long>(m) * m, 256), 256, 0, ctx->stream>>>(
        m, m, G, s->part.get(), ldp, a.part_stride, C, ldc);
    launched(ctx);
  }
  if (symmetric) {
    mirror_upper_kernel<<<grid_for(static_cast<long long>(m) * m, 256), 256, 0, ctx->stream>>>(m, C, ldc);
    launched(ctx);
  }
}

}  // namespace stgp

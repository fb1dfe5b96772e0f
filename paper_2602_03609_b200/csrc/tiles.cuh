// Tile-staged gathers (tiles.cu): outputs grouped into tiles of space-time neighbours whose
// source columns are staged once per M-chunk in shared memory.
#pragma once

#include <cstdint>

#include "common.cuh"

struct stgp_structure;

namespace stgp {

constexpr int kTileRows = 32;  // outputs per tile

struct TileSet {
  bool valid = false;
  int ntiles = 0, ucap = 0;  // tile count, largest union
  DevBuf<int32_t> tptr;   // ntiles + 1: outputs of tile t are out[tptr[t] .. tptr[t+1])
  DevBuf<int32_t> out;    // output indices (rows or columns) in locality order
  DevBuf<int32_t> uptr;   // ntiles + 1: union sources of tile t are ucol[uptr[t] .. uptr[t+1])
  DevBuf<int32_t> ucol;   // union source columns
  DevBuf<uint16_t> slot;  // (m_v + 1) union slots per output position (self last), 0xffff = none
};

struct TileSets {
  TileSet rows;
};

bool tiles_enabled();
void ensure_tiles(stgp_structure* s);
// Each returns false (nothing launched) when the tiled path does not apply; the caller then runs
// the per-row gather.
bool tile_vprime(stgp_structure* s, const double* W, const double* A, double* Vp);
bool tile_ef(stgp_structure* s, const double* W, const double* Rv, const double* c0, const double* D,
             const double* Vp, const double* yhat, const double* Bz, double* X_E, double* F);
bool tile_ga(stgp_structure* s, const double* W, const double* X, double* Ga);  // Ga: n x 32 (self at 31)

}  // namespace stgp

// bed_split_ws.cuh -- workspace shared by the three kernels of the medium
// path (bed_hh.cuh, bed_split.cuh).
#pragma once

#include "bed_common.cuh"

namespace bed {

// positions per record block: Q pads each sweep's record with identities to
// a whole block, F copies and applies whole blocks (one branch per block).  8
// at n = 64: fewer block joins, each of which costs the fold register moves
// (forward 8 192 x 64^2: 1.224 -> 1.174 ms); 4 below, where the padding costs
// more than the joins
template <int NMAX>
constexpr int fold_blk() { return NMAX >= 64 ? 8 : 4; }
constexpr int kQThreads = 32;  // one warp per CTA: small batches (n = 64) still reach every SM

struct SplitWs {
  float* P;         // [bc][n][n] initial V (VECS)
  float* D;         // [n][Bc] band diagonal, position-major
  float* E;         // [n][Bc] band off-diagonal
  float* lam;       // [n][Bc] unsorted eigenvalues (VECS)
  int32_t* vstat;   // [Bc] validation status from H
  float2* rot;      // [W][Smax][NMAX-1][32] recorded rotations (VECS)
  int32_t* msw;     // [W][Smax] warp-maximum active size of each recorded sweep
  int32_t* nsw;     // [W] sweeps recorded by warp w
  uint8_t* mlane;   // [W][Smax][32] each lane's active size in that sweep (0: no-op)
  int64_t Bc;       // chunk capacity (multiple of 32)
  int Smax;         // sweep records per warp
};

}  // namespace bed

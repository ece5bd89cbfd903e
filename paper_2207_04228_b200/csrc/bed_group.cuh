// bed_group.cuh -- lane-group communication for the row-parallel kernels.
//
// A matrix of order n <= NMAX is owned by a group of L lanes (L = 16 for
// NMAX <= 16, 32 for NMAX <= 32, 64 = two warps above that); lane r owns
// row r.  L <= 32: shuffles within the group's lanes.  L == 64: warp
// shuffles, then a two-slot exchange through shared memory ordered by a
// named barrier per group (ids 1..15).
#pragma once

#include "bed_common.cuh"

namespace bed {

template <int NMAX>
struct GroupSize {
  static constexpr int L = NMAX <= 16 ? 16 : (NMAX <= 32 ? 32 : 64);
};

template <int L>
struct Group {
  unsigned mask;  // lanes of this warp in the group
  int bar;        // named barrier id (L == 64)
  float* red;     // 4-word scratch (L == 64)
  int gl;         // lane in group

  __device__ __forceinline__ void init(int tid, int mi, float* scratch4) {
    const int lane = tid & 31;
    mask = L >= 32 ? 0xffffffffu : (((1u << L) - 1u) << (lane & ~(L - 1)));
    bar = 1 + mi;
    red = scratch4;
    gl = tid % L;
  }
  __device__ __forceinline__ void sync() const {
    if constexpr (L <= 32) __syncwarp(mask);
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(64) : "memory");
  }
  template <bool IS_MAX>
  __device__ __forceinline__ float reduce(float x) const {
    constexpr int W = L <= 32 ? L : 32;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      float y = __shfl_xor_sync(mask, x, o, W);
      x = IS_MAX ? fmaxf(x, y) : x + y;
    }
    if constexpr (L == 64) {
      if ((gl & 31) == 0) red[gl >> 5] = x;
      sync();
      x = IS_MAX ? fmaxf(red[0], red[1]) : red[0] + red[1];
      sync();
    }
    return x;
  }
  __device__ __forceinline__ float max(float x) const { return reduce<true>(x); }
  __device__ __forceinline__ float sum(float x) const { return reduce<false>(x); }
  // value held by group lane `src` (a compile-time constant at every call)
  __device__ __forceinline__ float bcast(float x, int src) const {
    if constexpr (L <= 32) {
      return __shfl_sync(mask, x, src, L);
    } else {
      if (gl == src) red[2] = x;
      sync();
      float res = red[2];
      sync();
      return res;
    }
  }
};

}  // namespace bed

// bed_tile.cuh -- CTA-cooperative copies between a batch of contiguous
// row-major n x n matrices in global memory and a padded shared stage laid
// out [matrix][row][col] (row stride SROW, matrix stride SMAT).
//
// The fast path (n == NMAX, n % 4 == 0, 16-byte aligned batch) moves
// 128-bit words and issues the loads of a batch of 8 words per thread
// before any shared store, so a thread has 8 global loads in flight instead
// of one dependent load per iteration.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bed {

// cp.async (Ampere+ LDGSTS): global -> shared without register staging.
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
// B in {4, 8, 16} bytes (both addresses B-aligned); larger B in 16-byte pieces
template <int B>
__device__ __forceinline__ void cp_async_bytes(void* sdst, const void* gsrc) {
  static_assert(B == 4 || B == 8 || B % 16 == 0, "cp.async moves 4, 8 or 16 bytes");
  if constexpr (B <= 16) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sdst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(s), "l"(gsrc), "n"(B) : "memory");
  } else {
#pragma unroll
    for (int o = 0; o < B; o += 16)
      cp_async_bytes<16>(static_cast<char*>(sdst) + o, static_cast<const char*>(gsrc) + o);
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int NMAX, int THREADS, int SROW, int SMAT>
__device__ __forceinline__ void tile_to_stage(const float* __restrict__ src, int count, int n,
                                              float* stage) {
  const int tid = threadIdx.x;
  if (n == NMAX && NMAX % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    constexpr int NN4 = NMAX * NMAX / 4;
    constexpr int B = 8;
    const int total = count * NN4;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    for (int base = 0; base < total; base += B * THREADS) {
      float4 buf[B];
#pragma unroll
      for (int q = 0; q < B; ++q) {
        const int i4 = base + tid + q * THREADS;
        buf[q] = i4 < total ? __ldg(s4 + i4) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      }
#pragma unroll
      for (int q = 0; q < B; ++q) {
        const int i4 = base + tid + q * THREADS;
        if (i4 < total) {
          const int mat = i4 / NN4, off = (i4 - mat * NN4) * 4;
          const int r = off / NMAX, c = off - r * NMAX;
          float* d = stage + mat * SMAT + r * SROW + c;
          if constexpr (SROW % 4 == 0 && SMAT % 4 == 0) {
            *reinterpret_cast<float4*>(d) = buf[q];
          } else {
            d[0] = buf[q].x; d[1] = buf[q].y; d[2] = buf[q].z; d[3] = buf[q].w;
          }
        }
      }
    }
  } else {
    const int nn = n * n;
#pragma unroll 4
    for (int g = tid; g < count * nn; g += THREADS) {
      const int mat = g / nn, off = g - mat * nn;
      const int r = off / n, c = off - r * n;
      stage[mat * SMAT + r * SROW + c] = __ldg(src + g);
    }
  }
}

// Asynchronous form of the fast path (cp.async, 16 bytes per copy): every
// word of the tile is in flight at once and no register holds it; the caller
// commits and waits (cp_async_commit / cp_async_wait_all + a barrier).
// Returns false when the fast path does not apply (the caller falls back).
template <int NMAX, int THREADS, int SROW, int SMAT>
__device__ __forceinline__ bool tile_to_stage_async(const float* __restrict__ src, int count, int n,
                                                    float* stage) {
  static_assert(SROW % 4 == 0 && SMAT % 4 == 0, "16-byte stage rows");
  if (!(n == NMAX && NMAX % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0)) return false;
  constexpr int NN4 = NMAX * NMAX / 4;
  const int total = count * NN4;
  for (int i4 = threadIdx.x; i4 < total; i4 += THREADS) {
    const int mat = i4 / NN4, off = (i4 - mat * NN4) * 4;
    const int r = off / NMAX, c = off - r * NMAX;
    cp_async_bytes<16>(stage + mat * SMAT + r * SROW + c, src + 4 * (int64_t)i4);
  }
  return true;
}

// The reverse copy; column c of matrix `mat` is multiplied by
// colscale[mat * NMAX + c] when colscale is given (sign normalisation).
template <int NMAX, int THREADS, int SROW, int SMAT>
__device__ __forceinline__ void stage_to_tile(const float* stage, int count, int n,
                                              float* __restrict__ dst,
                                              const float* colscale = nullptr) {
  const int tid = threadIdx.x;
  if (n == NMAX && NMAX % 4 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    constexpr int NN4 = NMAX * NMAX / 4;
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int i4 = tid; i4 < count * NN4; i4 += THREADS) {
      const int mat = i4 / NN4, off = (i4 - mat * NN4) * 4;
      const int r = off / NMAX, c = off - r * NMAX;
      const float* s = stage + mat * SMAT + r * SROW + c;
      float4 x = make_float4(s[0], s[1], s[2], s[3]);
      if (colscale) {
        const float* f = colscale + mat * NMAX + c;
        x.x *= f[0]; x.y *= f[1]; x.z *= f[2]; x.w *= f[3];
      }
      d4[i4] = x;
    }
  } else {
    const int nn = n * n;
    for (int g = tid; g < count * nn; g += THREADS) {
      const int mat = g / nn, off = g - mat * nn;
      const int r = off / n, c = off - r * n;
      float x = stage[mat * SMAT + r * SROW + c];
      if (colscale) x *= colscale[mat * NMAX + c];
      dst[g] = x;
    }
  }
}

}  // namespace bed

// bed_tc.cuh -- tcgen05 building blocks shared by the tensor-core kernels
// (bed_backward_tc.cuh, bed_power_tc.cuh): the K-major no-swizzle operand
// layout, shared-memory and instruction descriptors for kind::tf32 64 x 64 x 8
// MMAs, the 3xTF32 split, fences and TMEM loads.
#pragma once

#include <cstdint>

#include "bed_mbar.cuh"

namespace bed {

// byte offset of element (row, k) in a K-major no-swizzle operand
__device__ __forceinline__ uint32_t kmaj_off(int row, int k) {
  return (uint32_t)((row >> 3) * 2048 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

// x rounded to TF32 (10 explicit mantissa bits, to nearest).  The 3xTF32 split
// x = hi + lo uses it for both parts: hi = tf32(x), lo = tf32(x - hi), so the
// tensor core reads both exactly and what is dropped (|.| <= 2^-22 |x|) has no
// bias -- truncation would bias every product the same way, which adds up over
// long sums (the covariance producer's sample axis).
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// shared-memory matrix descriptor, version 1 (sm_100), no swizzle, K-major:
// LBO = 128 B (the next 4 k), SBO = 2048 B (the next 8 rows).  (MN-major
// descriptors, which would read the transposes from the same rows, gave no
// products for kind::tf32 in tools/ubench/umma_probe.cu, so the transposed
// operands are staged as such.)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | ((uint64_t)1 << 46);
}

// kind::tf32, D = F32, A/B = TF32 (K-major), M = 64, N = 64
constexpr uint32_t kIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((64u >> 4) << 24);
constexpr uint32_t kIdescTf32MN = kIdescTf32 | (1u << 15) | (1u << 16);  // probe only

__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc,
                                          uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void proxy_fence_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 16 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = __uint_as_float(r[q]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 8 values of an operand row (K-major), hi and lo, as two 16-byte chunks
__device__ __forceinline__ void store8(uint8_t* hi, uint8_t* lo, int row, int k0, const float (&d)[8]) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    float4 xh, xl;
    xh.x = tf32_hi(d[4 * q]);
    xh.y = tf32_hi(d[4 * q + 1]);
    xh.z = tf32_hi(d[4 * q + 2]);
    xh.w = tf32_hi(d[4 * q + 3]);
    xl = make_float4(tf32_hi(d[4 * q] - xh.x), tf32_hi(d[4 * q + 1] - xh.y), tf32_hi(d[4 * q + 2] - xh.z),
                     tf32_hi(d[4 * q + 3] - xh.w));
    const uint32_t o = kmaj_off(row, k0 + 4 * q);
    *reinterpret_cast<float4*>(hi + o) = xh;
    *reinterpret_cast<float4*>(lo + o) = xl;
  }
}

// M = 64 rows sit in TMEM lanes 0-15 of each subpartition: after a 16-column
// load, lane l (< 16) keeps columns 0-7 and lane l + 16 takes columns 8-15 of
// the same row, so all 32 lanes share the epilogue work
__device__ __forceinline__ void split_half(const float (&d)[16], int lane, float (&e)[8]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float up = __shfl_sync(0xffffffffu, d[8 + j], lane & 15);
    e[j] = lane < 16 ? d[j] : up;
  }
}

}  // namespace bed

// bed_f32x2.cuh -- packed FP32 pairs (sm_100a FFMA2 / FMUL2 / FADD2).
//
// Blackwell issues `fma.rn.f32x2` as one instruction carrying two FP32 FMAs
// (SASS FFMA2), with free operand swizzles: either half of a pair, or a
// scalar broadcast (`R.F32`), and per-half negation.  The FP32 pipe rate is
// unchanged (measured on B200: 71 TFLOP/s scalar FFMA, 73.7 TFLOP/s FFMA2,
// tools/ubench/ffma_peak.cu), so packing pays where a kernel is limited by
// instruction issue rather than by the FMA pipe -- the rotation folds and
// Householder updates here, which interleave FP work with selects, compares
// and shared-memory traffic.  Rounding is identical to the scalar ops
// (round-to-nearest, no contraction changes).
#pragma once

#include <cuda_runtime.h>

namespace bed {

struct f2 {
  unsigned long long r;
};

__device__ __forceinline__ f2 f2_make(float lo, float hi) {
  f2 o;
  asm("mov.b64 %0, {%1, %2};" : "=l"(o.r) : "f"(lo), "f"(hi));
  return o;
}
__device__ __forceinline__ f2 f2_bc(float x) { return f2_make(x, x); }
__device__ __forceinline__ float f2_lo(f2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.r));
  return x;
}
__device__ __forceinline__ float f2_hi(f2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.r));
  return y;
}
// a * b + c, per half
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
  f2 o;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(o.r) : "l"(a.r), "l"(b.r), "l"(c.r));
  return o;
}
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
  f2 o;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
  f2 o;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}

// Rotation of a column pair held as packed row pairs: with X = (x_r, x_r+1)
// and Y = (y_r, y_r+1) the entries of columns p and p+1 on two rows,
//   X <- c X - s Y,   Y <- s X + c Y        (_kernels.py:269-277)
// in four packed instructions for two rows.  ns = -s.
__device__ __forceinline__ void rot2(f2& X, f2& Y, float c, float s, float ns) {
  const f2 x = X, y = Y;
  X = ffma2(x, f2_bc(c), fmul2(y, f2_bc(ns)));
  Y = ffma2(x, f2_bc(s), fmul2(y, f2_bc(c)));
}

// rot2 written as one in-place asm block (the same four packed operations,
// same rounding): the outputs reuse the input registers, which keeps the
// register allocator from inserting moves at the joins of conditionally
// executed rotation blocks (bed_fold_tma.cuh).
__device__ __forceinline__ void rot2_ip(f2& X, f2& Y, float c, float s, float ns) {
  asm("{\n\t.reg .b64 t1, t2, cc, ss, nn;\n\t"
      "mov.b64 cc, {%2, %2};\n\tmov.b64 ss, {%3, %3};\n\tmov.b64 nn, {%4, %4};\n\t"
      "mul.rn.f32x2 t1, %1, nn;\n\t"
      "mul.rn.f32x2 t2, %1, cc;\n\t"
      "fma.rn.f32x2 %1, %0, ss, t2;\n\t"
      "fma.rn.f32x2 %0, %0, cc, t1;\n\t}"
      : "+l"(X.r), "+l"(Y.r)
      : "f"(c), "f"(s), "f"(ns));
}

}  // namespace bed

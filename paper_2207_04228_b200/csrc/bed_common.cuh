// bed_common.cuh -- scalar building blocks shared by the forward kernels.
//
// Each helper restates one reference primitive in FP32 (the reference is
// float64 numba; /root/reference/pkg/src/batchedeig/...):
//   givens()     rotation generation of _sweep_block, _kernels.py:244-258
//                (zero target -> identity rotation exactly, :247, :256-258)
//   wilkinson()  _wilkinson_scalar, _kernels.py:205-218 (mu_hi is the root
//                nearer the trailing entry, applied first: qr.py:67-76)
//   pow2_ceil()  _band_scale, qr.py:522-534 (exact power-of-two equilibration)
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <string.h>

#include <type_traits>

#define BED_HD __host__ __device__ __forceinline__

namespace bed {

constexpr int kStatusOk = 0;
constexpr int kStatusNoConv = 1;
constexpr int kStatusNonFinite = 2;
constexpr int kStatusNonSym = 3;
constexpr int kStatusNonPositive = 4;

// Column tails at or below this are already reduced (householder.py:37-39
// uses 1e-300 in float64; this is the FP32 analogue, well above the
// denormal range so 1/scale stays finite).
constexpr float kZeroTail = 1e-30f;

// Optional per-matrix diagnostics (the reference's SolveDiagnostics counters,
// qr.py:101-118, _kernels.py:396-398, per matrix): diag[3 j + 0] rotations
// applied (sum of active - 1 over the matrix's sweeps), [3 j + 1] reduction
// events (trailing deflations), [3 j + 2] step_r_sum (reductions so far,
// summed over its double steps); resid[j] the largest active coupling left
// when the step budget ran out (0 otherwise; NoConvergence's
// residual_offdiag_max, qr.py:385-389).  Either pointer may be null.
struct DiagOut {
  int32_t* diag;
  float* resid;
  __device__ __forceinline__ void put(int64_t j, int rot, int red, int srs, float res) const {
    if (diag) {
      diag[3 * j] = rot;
      diag[3 * j + 1] = red;
      diag[3 * j + 2] = srs;
    }
    if (resid) resid[j] = res;
  }
};

// f(x) = x^p of the spectral power (matrix_power, solver.py:115-143), exact
// for the common powers.
__device__ __forceinline__ float spectral_pow(float x, float p) {
  if (p == 1.0f) return x;
  if (p == 2.0f) return x * x;
  if (p == 0.5f) return sqrtf(x);
  if (p == -0.5f) return 1.0f / sqrtf(x);
  if (p == -1.0f) return 1.0f / x;
  return powf(x, p);
}

// Spectral power fused into the forward (bed_forward_power_f32): out =
// V diag(max(lambda, floor)^p) V^T instead of V.  floor_abs < 0 selects the
// reference default 1e-12 * lambda_max per matrix (solver.py:131-132).
struct PowSpec {
  float p;
  float floor_abs;
  int needs_positive;  // p negative or fractional: a non-positive clamped eigenvalue is an error
};

// Covariance producer fused in front of the forward (bed_scatter_forward_f32):
// the matrix is formed from X (batch, n, m) as (X - mu)(X - mu)^T + eps I
// (zca_whiten's scatter, solver.py:161-166) instead of being read.
struct ScatSpec {
  const float* X;
  int m;
  float eps;
};

struct KernelCfg {
  float eps;       // deflation_tol
  float sym_tol;   // symmetry_tol
  int max_steps;   // resolved double-step budget
  int sort;        // 0 none, 1 descending, 2 ascending
};

BED_HD float rsqrt_approx(float x) {
#ifdef __CUDA_ARCH__
  float y;  // one MUFU.RSQ; inputs here are normal numbers (no denormal fixup)
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#else
  return 1.0f / sqrtf(x);
#endif
}

// 1/sqrt(x) refined by one Newton step (MUFU.RSQ is ~2 ulp; the refined
// value keeps c^2 + s^2 within an ulp of 1 so V stays orthogonal over the
// thousands of rotations an n=64 solve folds).
BED_HD float rsqrt_nr(float x) {
  float y = rsqrt_approx(x);
  float hx = 0.5f * x;
  return y * fmaf(-hx * y, y, 1.5f);
}

// Givens rotation annihilating e against dw: R^T (dw, e) = (r, 0) with
// R = [[c, s], [-s, c]] (tests/helpers.py:14-22 convention, s = -e/r).
// A zero target gives the identity exactly (_kernels.py:247, :256-258); so
// does a target below 2^-60 of the equilibrated band (unit scale), which is
// far below FP32 resolution of any band entry it could couple.  With
// |e| >= 2^-60 the square sum is a normal number, so no scaled branch is
// needed (the reference's branch-scaled form, _kernels.py:248-258, guards
// float64 over/underflow that the equilibrated band cannot reach).
BED_HD void givens(float dw, float e, float& c, float& s, float& r) {
  const bool live = fabsf(e) >= 0x1p-60f;
  const float h2 = fmaf(dw, dw, e * e);
  const float ih = rsqrt_nr(h2);
  c = live ? dw * ih : 1.0f;
  s = live ? -e * ih : 0.0f;
  r = live ? h2 * ih : dw;
}

// Shift pair only (no rotation), fast math: the shifts steer convergence
// but every sweep is an exact similarity whatever their rounding, so they
// need not be correctly rounded.  hi is the root nearer d (applied first,
// qr.py:67-76); b == 0 gives (a, d) exactly like the reference shortcut.
BED_HD void wilkinson_shifts(float a, float b, float d, float& lo, float& hi) {
  const float h = 0.5f * (a - d);
  const float q = fmaf(h, h, b * b);
  const float rad = q > 0.0f ? q * rsqrt_approx(q) : 0.0f;
  const float mid = 0.5f * (a + d);
  const float nearer = h >= 0.0f ? mid - rad : mid + rad;
  const float farther = h >= 0.0f ? mid + rad : mid - rad;
  hi = b == 0.0f ? d : nearer;
  lo = b == 0.0f ? a : farther;
}

// Fast reciprocal (one MUFU.RCP): the reflector code only needs a ratio that
// is used consistently; normalisation happens afterwards with rsqrt_nr.
BED_HD float rcp_fast(float x) {
#ifdef __CUDA_ARCH__
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#else
  return 1.0f / x;
#endif
}

// Eigenvalue pair of [[a, b], [b, d]] plus its diagonalising rotation.
BED_HD void wilkinson(float a, float b, float d, float& lo, float& hi, float& c, float& s) {
  if (b == 0.0f) {
    lo = a;
    hi = d;
    c = 1.0f;
    s = 0.0f;
    return;
  }
  float m = (a - d) / (2.0f * b);
  float sign = m >= 0.0f ? 1.0f : -1.0f;
  float am = fabsf(m);
  float root = am > 1e18f ? am : sqrtf(fmaf(m, m, 1.0f));  // hypot(1, m)
  float t = -sign / (am + root);
  c = 1.0f / sqrtf(fmaf(t, t, 1.0f));
  s = c * t;
  float bcs2 = 2.0f * b * c * s;
  lo = (a * c * c - bcs2) + d * s * s;
  hi = (a * s * s + bcs2) + d * c * c;
}

BED_HD float bits_to_float(int b) {
#ifdef __CUDA_ARCH__
  return __int_as_float(b);
#else
  float f;
  memcpy(&f, &b, sizeof f);
  return f;
#endif
}

// 2^ceil(log2(top)) for top > 0 (1 for top == 0), computed exactly from the
// exponent bits; returns the power and its exact inverse.
BED_HD float pow2_ceil(float top, float* inv = nullptr) {
  float p = 1.0f, ip = 1.0f;
  if (top > 0.0f && top <= 0x1p126f) {
    int ex;
    const float f = frexpf(top, &ex);  // top = f * 2^ex, f in [0.5, 1)
    if (f == 0.5f) ex -= 1;
    ex = ex < -125 ? -125 : ex;
    p = bits_to_float((ex + 127) << 23);
    ip = bits_to_float((127 - ex) << 23);
  } else if (top > 0x1p126f) {
    p = 0x1p127f;
    ip = 0x1p-127f;
  }
  if (inv) *inv = ip;
  return p;
}

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).  Used
// where a loop index must be a constant so register arrays stay in
// registers -- the NVVM unroller gives up on very large bodies (the n = 64
// reduction), template expansion never does.
template <int B, int E, typename F>
BED_HD void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Stable rank of slot c among n values for the requested order: the
// position _sort_and_sign (solver.py:60-76) moves slot c to.
BED_HD bool rank_before(float kv, int kidx, float v, int idx, int sort) {
  // does (kv, kidx) sort strictly before (v, idx)?
  if (sort == 1) return kv > v || (kv == v && kidx < idx);
  return kv < v || (kv == v && kidx < idx);
}

}  // namespace bed

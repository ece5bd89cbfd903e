// bed_scatter_regs.cuh -- the covariance producer for n <= 8 with one thread
// per matrix: the thread streams its own n x m block
// of X once (128-bit loads along samples when rows allow) and keeps the lower
// triangle of the scatter, the channel sums and the shift in registers.
//
// Used by the fused covariance -> ED path (bed_small_kernel<..., SCAT>), where
// the matrix goes straight into the solver's registers, and by the standalone
// producer below for n <= 8 (the tiled bed_scatter_kernel's per-CTA staging
// costs more than the data at these sizes: 1M x 4 x 16 took 1.4 ms).
//
// Formula (as bed_scatter.cu): one pass shifted by each channel's first
// sample x0,  S = sum_k (x_k - x0)(x_k - x0)^T - m d d^T,  d = mean(x - x0),
// then + eps I -- the reference zca_whiten's (X - mu)(X - mu)^T + eps I
// (solver.py:161-166); exactly symmetric by construction.
#pragma once
#include <cstdint>

#include "bed_common.cuh"

namespace bed {

template <int N>
__device__ __forceinline__ void scatter_regs(const float* __restrict__ xr, int m, float eps,
                                             bool live, bool aligned16, float (&x)[N][N]) {
  float x0[N], sum[N], s[N][N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    x0[r] = live ? __ldg(xr + (int64_t)r * m) : 0.0f;
    sum[r] = 0.0f;
#pragma unroll
    for (int c = 0; c <= r; ++c) s[r][c] = 0.0f;
  }
  auto acc = [&](const float (&y)[N]) {
#pragma unroll
    for (int r = 0; r < N; ++r) {
      sum[r] += y[r];
#pragma unroll
      for (int c = 0; c <= r; ++c) s[r][c] = fmaf(y[r], y[c], s[r][c]);
    }
  };
  int k = 0;
  if (live && m % 4 == 0 && aligned16) {
    for (; k < m; k += 4) {
      float4 t[N];
#pragma unroll
      for (int r = 0; r < N; ++r) t[r] = __ldg(reinterpret_cast<const float4*>(xr + (int64_t)r * m + k));
      float y[N];
#pragma unroll
      for (int r = 0; r < N; ++r) y[r] = t[r].x - x0[r];
      acc(y);
#pragma unroll
      for (int r = 0; r < N; ++r) y[r] = t[r].y - x0[r];
      acc(y);
#pragma unroll
      for (int r = 0; r < N; ++r) y[r] = t[r].z - x0[r];
      acc(y);
#pragma unroll
      for (int r = 0; r < N; ++r) y[r] = t[r].w - x0[r];
      acc(y);
    }
  }
  for (; live && k < m; ++k) {
    float y[N];
#pragma unroll
    for (int r = 0; r < N; ++r) y[r] = __ldg(xr + (int64_t)r * m + k) - x0[r];
    acc(y);
  }
  const float fm = (float)m;
#pragma unroll
  for (int r = 0; r < N; ++r) sum[r] = sum[r] / fm;
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) {
      const float v = fmaf(-fm * sum[r], sum[c], s[r][c]) + (r == c ? eps : 0.0f);
      x[r][c] = live ? v : 0.0f;
      x[c][r] = x[r][c];
    }
}

constexpr int kScatSmallThreads = 128;

// Standalone producer, n <= 8: thread j forms matrix base + j in registers and
// parks it in shared memory at an odd per-matrix stride (conflict-free); the
// CTA's 128 matrices then leave as one contiguous, coalesced block.
template <int N>
__global__ void __launch_bounds__(kScatSmallThreads)
    bed_scatter_small_kernel(const float* __restrict__ X, float* __restrict__ out, int64_t batch,
                             int m, float eps) {
  constexpr int NN = N * N, STRIDE = NN | 1;
  __shared__ float stage[kScatSmallThreads * STRIDE];
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kScatSmallThreads;
  const bool live = base + tid < batch;
  float x[N][N];
  scatter_regs<N>(X + (base + (live ? tid : 0)) * (int64_t)N * m, m, eps, live,
                  (reinterpret_cast<uintptr_t>(X) & 15) == 0, x);
#pragma unroll
  for (int r = 0; r < N; ++r)
#pragma unroll
    for (int c = 0; c < N; ++c) stage[tid * STRIDE + r * N + c] = x[r][c];
  __syncthreads();
  const int64_t left = batch - base;
  const int count = left < kScatSmallThreads ? (int)left : kScatSmallThreads;
  float* o = out + base * NN;
  for (int g = tid; g < count * NN; g += kScatSmallThreads) {
    const int mat = g / NN;
    o[g] = stage[mat * STRIDE + (g - mat * NN)];
  }
}

}  // namespace bed

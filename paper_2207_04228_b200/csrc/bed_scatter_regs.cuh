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

// Warp-staged form (m % 8 == 0, 32-byte aligned X): the same sums, but X
// reaches the threads through a per-warp shared stage, 8 samples at a time.
// Each 128-bit load takes half of one (matrix, channel) 32-byte segment, so a
// warp's request covers 16 whole sectors -- the per-thread form above makes
// every request touch 32 half-used sectors, which left the L1 95 % busy and
// refetched each sector from L2 (ncu, 1 M x 4 x 16).  Stage stride 8N + 4
// floats per matrix: conflict-free 128-bit stores and loads.
template <int N>
struct ScatStage {
  static constexpr int KC = 8;                 // samples per stage
  static constexpr int MS = KC * N + 4;        // floats per matrix
  static constexpr int WARP = 32 * MS;         // floats per warp
};

template <int N>
__device__ __forceinline__ void scatter_regs_staged(const float* __restrict__ xw, int nlive, int m,
                                                    float eps, int lane, float* __restrict__ xs,
                                                    float (&x)[N][N]) {
  using S = ScatStage<N>;
  const bool live = lane < nlive;
  float x0[N], sum[N], s[N][N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
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
  const float* mine = xs + lane * S::MS;
  for (int k0 = 0; k0 < m; k0 += S::KC) {
    // 32 N segments of 8 samples, two lanes per segment, 16 segments per step
#pragma unroll
    for (int q = 0; q < 2 * N; ++q) {
      const int sg = 16 * q + (lane >> 1), half = lane & 1;
      const int mat = sg / N, row = sg - mat * N;
      float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (mat < nlive) v = __ldg(reinterpret_cast<const float4*>(xw + ((int64_t)mat * N + row) * m + k0) + half);
      *reinterpret_cast<float4*>(xs + mat * S::MS + row * S::KC + 4 * half) = v;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // four samples of every row at a time (register pressure)
      float xv[N][4];
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const float4 a = *reinterpret_cast<const float4*>(mine + r * S::KC + 4 * h);
        xv[r][0] = a.x; xv[r][1] = a.y; xv[r][2] = a.z; xv[r][3] = a.w;
      }
      if (k0 == 0 && h == 0) {
#pragma unroll
        for (int r = 0; r < N; ++r) x0[r] = xv[r][0];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float y[N];
#pragma unroll
        for (int r = 0; r < N; ++r) y[r] = xv[r][j] - x0[r];
        acc(y);
      }
    }
    __syncwarp();  // the stage is refilled next step
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

// X's rows can be read in 8-sample, 32-byte segments
__host__ __device__ inline bool scatter_staged_ok(const float* X, int m) {
  return m % 8 == 0 && (reinterpret_cast<uintptr_t>(X) & 31) == 0;
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
  constexpr int XS = 4 * ScatStage<N>::WARP;
  constexpr int SMEM = XS > kScatSmallThreads * STRIDE ? XS : kScatSmallThreads * STRIDE;
  __shared__ __align__(16) float stage[SMEM];  // X stage (per warp), then S for the stores
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kScatSmallThreads;
  const bool live = base + tid < batch;
  float x[N][N];
  if (scatter_staged_ok(X, m)) {
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t wbase = base + 32 * warp;
    const int64_t wl = batch - wbase;
    const int nlive = wl <= 0 ? 0 : (wl < 32 ? (int)wl : 32);
    scatter_regs_staged<N>(X + (nlive > 0 ? wbase : 0) * (int64_t)N * m, nlive, m, eps, lane,
                           stage + warp * ScatStage<N>::WARP, x);
    __syncthreads();  // the X stage becomes the S stage
  } else {
    scatter_regs<N>(X + (base + (live ? tid : 0)) * (int64_t)N * m, m, eps, live,
                    (reinterpret_cast<uintptr_t>(X) & 15) == 0, x);
  }
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

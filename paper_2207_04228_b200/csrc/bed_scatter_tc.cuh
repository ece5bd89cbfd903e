// bed_scatter_tc.cuh -- the covariance producer (bed_scatter.cu) for
// 33 <= n <= 64 on the tcgen05 tensor cores in 3xTF32 (bed_tc.cuh):
//   S = sym( Y Y^T - m d d^T ) + eps I,   Y = X - x0,  d = rowsum(Y) / m
// -- the scatter of the reference zca_whiten (solver.py:161-166), the one-pass
// shifted formula of bed_scatter.cu, here shifted by each channel's mean over
// its first 64 samples: Y Y^T and m d d^T then nearly cancel only by the
// sampling error of that mean, which the tensor core's (3xTF32) rounding
// needs -- a first-sample shift left 2e-5 relative error at n = 64, m = 256.  Y Y^T is one product with A = B
// = Y (both Y's rows, K = samples), accumulated in TMEM over chunks of 64
// samples; each chunk's loads are issued while the previous chunk's MMAs run.
// The per-channel sums are kept in registers by the threads that stage Y and
// reduced in a fixed order (deterministic).  S goes through a padded shared
// stage for the exact symmetrisation (solver.py:164).
#pragma once

#include "bed_common.cuh"
#include "bed_tc.cuh"

namespace bed {

struct ScatTcParams {
  static constexpr int THREADS = 256;
  static constexpr int BUF = 64 * 64 * 4;       // one 64-sample chunk of Y (hi or lo)
  static constexpr int OFF_PART = 2 * BUF;      // row-sum partials [4][64], x0 [64], d [64]
  static constexpr int OFF_BAR = OFF_PART + 6 * 64 * 4;
  static constexpr int OFF_TMEM = OFF_BAR + 8;
  static constexpr size_t BYTES = OFF_TMEM + 8;
  static constexpr int CTAS_PER_SM = 4;
  static constexpr int SPITCH = 65;             // S stage row pitch (in the Y region)
  static_assert(64 * SPITCH * 4 <= 2 * BUF, "stage fits in the chunk buffer");
};

__global__ void __launch_bounds__(ScatTcParams::THREADS, ScatTcParams::CTAS_PER_SM)
    bed_scatter_tc_kernel(const float* __restrict__ X, float* __restrict__ out, int64_t batch, int n,
                          int m, float eps) {
  using P = ScatTcParams;
  extern __shared__ __align__(1024) uint8_t sc_smem[];
  uint8_t* const smem = sc_smem;
  uint8_t* const y_hi = smem;
  uint8_t* const y_lo = smem + P::BUF;
  float* sPart = reinterpret_cast<float*>(smem + P::OFF_PART);  // [4][64]
  float* sX0 = sPart + 4 * 64;
  float* sD = sX0 + 64;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + P::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::OFF_TMEM);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  uint32_t phase = 0;
  const int nn = n * n;
  const int64_t per = (int64_t)n * m;
  const int nchunk = (m + 63) / 64;
  const int sub = warp & 3, ch = warp >> 2;
  const int r = 16 * sub + (lane & 15);
  const int c_lo = 32 * ch;
  const int c_half = lane < 16 ? 0 : 8;
  const uint32_t trow = tmem + ((uint32_t)(32 * sub) << 16) + (uint32_t)c_lo;
  const bool vec4 = (m % 4 == 0) && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  // staging geometry: step u covers core block c = warp + 8u: rows 8 rb + lane % 8,
  // sample group 4 kq + lane / 8 of the chunk; rows (and so the row-sum
  // partials) are fixed per thread
  auto srow = [&](int u) { return 8 * ((warp + 8 * u) >> 2) + (lane & 7); };
  const int kq = warp & 3;
  const int k0 = 4 * (4 * kq + (lane >> 3));  // sample offset within a chunk

  float4 px[4];
  auto prefetch = [&](int64_t mm, int chunk) {
    const bool have = mm < batch;
    const float* xb = X + (have ? mm : 0) * per;
    const int s0 = 64 * chunk + k0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int row = srow(u);
      px[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (have && row < n && s0 < m) {
        const float* src = xb + (int64_t)row * m + s0;
        if (vec4) {
          px[u] = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          px[u].x = __ldg(src);
          px[u].y = s0 + 1 < m ? __ldg(src + 1) : 0.0f;
          px[u].z = s0 + 2 < m ? __ldg(src + 2) : 0.0f;
          px[u].w = s0 + 3 < m ? __ldg(src + 3) : 0.0f;
        }
      }
    }
  };

  prefetch(blockIdx.x, 0);
  for (int64_t mm = blockIdx.x; mm < batch; mm += gridDim.x) {
    // shift: each channel's mean over the first chunk (up to 64 samples), from
    // the prefetched chunk, reduced in a fixed order like the sums below
    float x0[4], rs[4];
    {
      const int s0 = k0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float v = (s0 < m ? px[u].x : 0.0f) + (s0 + 1 < m ? px[u].y : 0.0f);
        v += (s0 + 2 < m ? px[u].z : 0.0f) + (s0 + 3 < m ? px[u].w : 0.0f);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (lane < 8) sPart[kq * 64 + srow(u)] = v;
      }
      __syncthreads();
      if (tid < 64)
        sX0[tid] = (((sPart[tid] + sPart[64 + tid]) + sPart[128 + tid]) + sPart[192 + tid]) / (float)(m < 64 ? m : 64);
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x0[u] = sX0[srow(u)];
        rs[u] = 0.0f;
      }
    }
    for (int chunk = 0; chunk < nchunk; ++chunk) {
      // ---- stage Y = X - x0 for this chunk (samples past m are zero), hi/lo
      const int s0 = 64 * chunk + k0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = srow(u);
        const bool rv = row < n;
        float4 y;
        y.x = (rv && s0 < m) ? px[u].x - x0[u] : 0.0f;
        y.y = (rv && s0 + 1 < m) ? px[u].y - x0[u] : 0.0f;
        y.z = (rv && s0 + 2 < m) ? px[u].z - x0[u] : 0.0f;
        y.w = (rv && s0 + 3 < m) ? px[u].w - x0[u] : 0.0f;
        rs[u] += (y.x + y.y) + (y.z + y.w);
        const float4 h = make_float4(tf32_hi(y.x), tf32_hi(y.y), tf32_hi(y.z), tf32_hi(y.w));
        const uint32_t o = kmaj_off(row, k0);
        *reinterpret_cast<float4*>(y_hi + o) = h;
        *reinterpret_cast<float4*>(y_lo + o) = make_float4(tf32_hi(y.x - h.x), tf32_hi(y.y - h.y), tf32_hi(y.z - h.z),
                                                                tf32_hi(y.w - h.w));
      }
      proxy_fence_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const uint32_t hi = smem_u32(y_hi), lo = smem_u32(y_lo);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t o = 256u * kk;
          umma_tf32(tmem, umma_desc(lo + o, 128u, 2048u), umma_desc(hi + o, 128u, 2048u), kIdescTf32,
                    (chunk > 0 || kk > 0) ? 1u : 0u);
          umma_tf32(tmem, umma_desc(hi + o, 128u, 2048u), umma_desc(lo + o, 128u, 2048u), kIdescTf32, 1u);
          umma_tf32(tmem, umma_desc(hi + o, 128u, 2048u), umma_desc(hi + o, 128u, 2048u), kIdescTf32, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(bar))
                     : "memory");
      }
      // the next chunk (or the next matrix's first) is loaded while the MMAs run
      if (chunk + 1 < nchunk) prefetch(mm, chunk + 1);
      else prefetch(mm + gridDim.x, 0);
      mbar_wait(bar, phase);
      phase ^= 1;
      tc_fence_after();
    }
    // ---- d = rowsum(Y) / m, reduced in a fixed order: lanes l, l+8, l+16,
    // l+24 share a row (shuffle), the four warps w % 4 = kq by index
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float v = rs[u];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (lane < 8) sPart[kq * 64 + srow(u)] = v;
    }
    __syncthreads();
    const float fm = (float)m;
    if (tid < 64) sD[tid] = (((sPart[tid] + sPart[64 + tid]) + sPart[128 + tid]) + sPart[192 + tid]) / fm;
    __syncthreads();
    // ---- S = D - m d d^T through the stage (the Y region: all MMAs are done)
    float* sg = reinterpret_cast<float*>(y_hi);
    const float dr = sD[r] * fm;
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      float d[16], e[8];
      tmem_ld16(trow + 16u * q, d);
      tmem_wait_ld();
      split_half(d, lane, e);
      const int cb = c_lo + 16 * q + c_half;
#pragma unroll
      for (int j = 0; j < 8; ++j) sg[r * P::SPITCH + cb + j] = fmaf(-dr, sD[cb + j], e[j]);
    }
    tc_fence_before();
    __syncthreads();
    for (int rr = warp; rr < n; rr += P::THREADS / 32) {
      float* dst = out + mm * nn + rr * n;
      const float* grow = sg + rr * P::SPITCH;
      const float* gcol = sg + rr;
      float v = 0.5f * (grow[lane] + gcol[lane * P::SPITCH]);  // n > 32
      dst[lane] = lane == rr ? v + eps : v;
      if (lane + 32 < n) {
        v = 0.5f * (grow[lane + 32] + gcol[(lane + 32) * P::SPITCH]);
        dst[lane + 32] = lane + 32 == rr ? v + eps : v;
      }
    }
    __syncthreads();  // the stage is the next matrix's Y buffer
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

}  // namespace bed

// bed_power_tc.cuh -- the spectral power  out = sym( V diag(f) V^T ),
// f_k = max(lambda_k, floor)^p  (matrix_power, solver.py:115-143), for
// 33 <= n <= 64 on the tcgen05 tensor cores in 3xTF32 -- the machinery of
// bed_backward_tc.cuh (bed_tc.cuh: 64 x 64 x 8 MMAs, TMEM accumulator).
//
// One product per matrix and no transposes: A = V diag(f) (row i = V[i][k] f_k)
// and B = V (row j = V[j][k]) are both V's rows, so D = A B^T = V diag(f) V^T.
// The floor, the positivity rule and the merge semantics are those of
// bed_power.cu; D goes through a padded shared stage so the output is
// (D + D^T) / 2 exactly symmetric, like the reference (solver.py:141).
// A CTA (8 warps, three per SM) works on one matrix at a time, persistent;
// the next matrix's V is loaded while the current product runs.
#pragma once

#include "bed_common.cuh"
#include "bed_tc.cuh"

namespace bed {

struct PowTcParams {
  static constexpr int THREADS = 256;
  static constexpr int BUF = 64 * 64 * 4;       // one operand copy (hi or lo)
  static constexpr int OFF_F = 4 * BUF;         // A hi, A lo, B hi, B lo; then f[64]
  static constexpr int OFF_BAR = OFF_F + 64 * 4;
  static constexpr int OFF_TMEM = OFF_BAR + 8;
  static constexpr size_t BYTES = OFF_TMEM + 8;
  static constexpr int CTAS_PER_SM = 3;
  static constexpr int SPITCH = 65;             // D stage row pitch (in the A region)
  static_assert(64 * SPITCH * 4 <= 2 * BUF, "stage fits in A");
};

__global__ void __launch_bounds__(PowTcParams::THREADS, PowTcParams::CTAS_PER_SM)
    bed_power_tc_kernel(const float* __restrict__ V, const float* __restrict__ lam,
                        float* __restrict__ out, int32_t* __restrict__ status,
                        int32_t* __restrict__ flags, int64_t batch, int n, float p, float floor_abs,
                        int needs_positive, int merge) {
  using P = PowTcParams;
  extern __shared__ __align__(1024) uint8_t pw_smem[];
  uint8_t* const smem = pw_smem;
  uint8_t* const a_hi = smem;
  uint8_t* const a_lo = smem + P::BUF;
  uint8_t* const b_hi = smem + 2 * P::BUF;
  uint8_t* const b_lo = smem + 3 * P::BUF;
  float* sF = reinterpret_cast<float*>(smem + P::OFF_F);
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
  const int sub = warp & 3, ch = warp >> 2;
  const int r = 16 * sub + (lane & 15);
  const int c_lo = 32 * ch;
  const int c_half = lane < 16 ? 0 : 8;
  const uint32_t trow = tmem + ((uint32_t)(32 * sub) << 16) + (uint32_t)c_lo;
  const bool vec4 = (n % 4 == 0) && (reinterpret_cast<uintptr_t>(V) & 15) == 0;

  // V's rows as 8-row x 4-k core blocks: lane -> (row 8 rb + lane % 8,
  // k-group 4 kq + lane / 8); 32 blocks per matrix, 4 per warp
  float4 pv[4];
  float pl = 0.0f;
  auto prefetch = [&](int64_t mm) {
    const bool have = mm < batch;
    const float* vb = V + (have ? mm : 0) * nn;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = warp + 8 * u;
      const int row = 8 * (c >> 2) + (lane & 7), k0 = 4 * (4 * (c & 3) + (lane >> 3));
      pv[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (have && row < n && k0 < n) {
        const float* src = vb + row * n + k0;
        if (vec4) {
          pv[u] = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          pv[u].x = __ldg(src);
          pv[u].y = k0 + 1 < n ? __ldg(src + 1) : 0.0f;
          pv[u].z = k0 + 2 < n ? __ldg(src + 2) : 0.0f;
          pv[u].w = k0 + 3 < n ? __ldg(src + 3) : 0.0f;
        }
      }
    }
    pl = (have && tid < n) ? __ldg(lam + mm * n + tid) : -INFINITY;
  };
  prefetch(blockIdx.x);
  for (int64_t m = blockIdx.x; m < batch; m += gridDim.x) {
    // ---- f (bed_power.cu): warps 0-1 hold the 64 eigenvalues
    if (tid < 64) sF[tid] = pl;
    __syncthreads();
    if (warp == 0) {
      const float l0 = sF[lane], l1 = sF[lane + 32];
      float lmax = fmaxf(l0, l1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lmax = fmaxf(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
      const float fl = floor_abs < 0.0f ? 1e-12f * lmax : floor_abs;
      const float x0 = fmaxf(l0, fl), x1 = fmaxf(l1, fl);
      const bool bad = __any_sync(0xffffffffu, needs_positive && ((lane < n && !(x0 > 0.0f)) ||
                                                                  (lane + 32 < n && !(x1 > 0.0f))));
      sF[lane] = (bad || lane >= n) ? 0.0f : spectral_pow(x0, p);
      sF[lane + 32] = (bad || lane + 32 >= n) ? 0.0f : spectral_pow(x1, p);
      if (lane == 0) {
        bool flag = bad;
        if (merge) flag = bad && (!status || status[m] == kStatusOk);
        if (status && (flag || !merge)) status[m] = flag ? kStatusNonPositive : kStatusOk;
        if (flag && flags) atomicOr(flags, 1 << kStatusNonPositive);
      }
    }
    __syncthreads();
    // ---- stage A = V diag(f), B = V, hi/lo
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = warp + 8 * u;
      const int row = 8 * (c >> 2) + (lane & 7), k0 = 4 * (4 * (c & 3) + (lane >> 3));
      const uint32_t o = kmaj_off(row, k0);
      const float4 v = pv[u];
      const float4 bh = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
      *reinterpret_cast<float4*>(b_hi + o) = bh;
      *reinterpret_cast<float4*>(b_lo + o) = make_float4(tf32_hi(v.x - bh.x), tf32_hi(v.y - bh.y), tf32_hi(v.z - bh.z),
                                                          tf32_hi(v.w - bh.w));
      const float4 a = make_float4(v.x * sF[k0], v.y * sF[k0 + 1], v.z * sF[k0 + 2], v.w * sF[k0 + 3]);
      const float4 ah = make_float4(tf32_hi(a.x), tf32_hi(a.y), tf32_hi(a.z), tf32_hi(a.w));
      *reinterpret_cast<float4*>(a_hi + o) = ah;
      *reinterpret_cast<float4*>(a_lo + o) = make_float4(tf32_hi(a.x - ah.x), tf32_hi(a.y - ah.y), tf32_hi(a.z - ah.z),
                                                          tf32_hi(a.w - ah.w));
    }
    proxy_fence_smem();
    tc_fence_before();
    __syncthreads();
    // ---- D = (V diag f) V^T
    if (tid == 0) {
      tc_fence_after();
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t o = 256u * kk;
        umma_tf32(tmem, umma_desc(al + o, 128u, 2048u), umma_desc(bh + o, 128u, 2048u), kIdescTf32,
                  kk > 0 ? 1u : 0u);
        umma_tf32(tmem, umma_desc(ah + o, 128u, 2048u), umma_desc(bl + o, 128u, 2048u), kIdescTf32, 1u);
        umma_tf32(tmem, umma_desc(ah + o, 128u, 2048u), umma_desc(bh + o, 128u, 2048u), kIdescTf32, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(bar))
                   : "memory");
    }
    prefetch(m + gridDim.x);  // the next matrix's V, in flight during the product
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    // ---- D through the stage (the A region), out = (D + D^T) / 2
    float* sg = reinterpret_cast<float*>(a_hi);
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      float d[16], e[8];
      tmem_ld16(trow + 16u * q, d);
      tmem_wait_ld();
      split_half(d, lane, e);
#pragma unroll
      for (int j = 0; j < 8; ++j) sg[r * P::SPITCH + c_lo + 16 * q + c_half + j] = e[j];
    }
    tc_fence_before();
    __syncthreads();
    for (int rr = warp; rr < n; rr += P::THREADS / 32) {
      float* dst = out + m * nn + rr * n;
      const float* grow = sg + rr * P::SPITCH;
      const float* gcol = sg + rr;
      dst[lane] = 0.5f * (grow[lane] + gcol[lane * P::SPITCH]);  // n > 32
      if (lane + 32 < n) dst[lane + 32] = 0.5f * (grow[lane + 32] + gcol[(lane + 32) * P::SPITCH]);
    }
    __syncthreads();  // stage and operands are rewritten for the next matrix
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

}  // namespace bed

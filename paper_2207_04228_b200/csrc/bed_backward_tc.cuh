// bed_backward_tc.cuh -- the Taylor-K ED backward for 33 <= n <= 64 on the
// 5th-generation tensor cores (tcgen05, accumulators in TMEM), in 3xTF32.
//
//   gA = sym( V (F o (V^T gV) + diag(gL)) V^T )      (bed_backward.cuh)
//
// Why 3xTF32: a single TF32 pass gives gradients 5-10e-4 off float64 (the gate
// is 1e-4); splitting every operand x = hi + lo (hi = x rounded to TF32,
// lo = x - hi rounded to TF32, bed_tc.cuh) and accumulating lo*hi + hi*lo +
// hi*hi gives ~1e-6 (tools/bwd_tc_check.py).
//
// A CTA (8 warps, three per SM) works on one matrix at a time, persistent over
// the batch, with 64 x 64 x 8 MMAs (cta_group::1, M = 64: row m of D sits in
// TMEM lane 32 (m / 16) + m % 16).  The three products are arranged so every
// intermediate leaves the epilogue in the row-per-thread orientation the next
// product reads:
//   P1  D = gV^T V   = M^T      A = gV^T, B = V^T (staged transposed from HBM)
//   E1  M'^T = (F o M + diag gL)^T, row by row            -> X1 (B of P2)
//   P2  D = V M'     = W        A = V (staged as is, in X2),  B = M'^T
//   E2  W, row by row                                      -> X1 (A of P3)
//   P3  D = W V^T    = G        A = W, B = V
//   E3  G through a padded shared stage, gA = (G + G^T) / 2, coalesced
// Operands live in shared memory in the canonical K-major no-swizzle layout
// (8-row x 16-byte core matrices; LBO = 128 B between the two core matrices
// of one K = 8 step, SBO = 2 KB between 8-row groups), each as hi and lo
// copies in two operand buffers (2 x 2 x 16 KB): X1 = gV^T -> M'^T -> W -> the
// G stage, X2 = V^T -> V (V's 128-bit loads are issued with P1, stored after
// E1, once P1 has read V^T), so three CTAs fit per SM.  One elected thread issues the 3 x 8 MMAs of
// a product and commits them to an mbarrier the CTA waits on.
#pragma once

#include <cstdint>

#include "bed_common.cuh"
#include "bed_tc.cuh"

namespace bed {

struct BwdTcParams {
  static constexpr int THREADS = 256;  // 8 warps: warps w and w + 4 share TMEM lanes, split columns
  static constexpr int BUF = 64 * 64 * 4;              // one operand copy (hi or lo), bytes
  static constexpr int OPS = 2;                        // X1 (gV^T -> M'^T -> W -> G stage), X2 (V^T -> V)
  static constexpr int OFF_LAM = OPS * 2 * BUF;        // lam[64], inv[64], gL[64]
  static constexpr int OFF_BAR = OFF_LAM + 3 * 64 * 4;
  static constexpr int OFF_TMEM = OFF_BAR + 8;
  static constexpr int OFF_OUT = OFF_TMEM + 8;
  static constexpr size_t BYTES = OFF_OUT + 16;
  static constexpr int CTAS_PER_SM = 3;
  static constexpr int SPITCH = 65;                    // G stage row pitch (floats)
  static_assert(64 * SPITCH * 4 <= 2 * BUF, "G stage fits in X1");
};

// one element of F (bed_backward.cuh): the Taylor series of 1/(l_j - l_i)
// about the pair's larger eigenvalue, the exact value outside its domain
// (CHECK = false when every eigenvalue of the pair is positive: always inside)
template <bool CHECK>
__device__ __forceinline__ float taylor_f(int i, int j, float li, float lj, float ii_inv, float ij_inv,
                                          int degree, int n, bool& off) {
  const bool hf = i < j ? (li >= lj) : (li > lj);
  const float binv = hf ? ii_inv : ij_inv;
  const float ratio = (hf ? lj : li) * binv;
  float poly = 1.0f;
  if (degree == 9) {  // the paper's degree, unrolled
#pragma unroll
    for (int k = 0; k < 9; ++k) poly = fmaf(poly, ratio, 1.0f);
  } else {
    for (int k = 0; k < degree; ++k) poly = fmaf(poly, ratio, 1.0f);
  }
  float tv = poly * binv;
  if constexpr (CHECK) {
    const float big = hf ? li : lj, small = hf ? lj : li;
    const bool in_domain = (big > 0.0f && (fabsf(ratio) < 1.0f || small == big)) ||
                           (big == 0.0f && small == 0.0f);
    if (!in_domain && i != j && i < n && j < n) {
      tv = big != small ? 1.0f / (big - small) : 0.0f;
      off = true;
    }
  }
  return i == j ? 0.0f : (hf ? -tv : tv);
}

__global__ void __launch_bounds__(BwdTcParams::THREADS, BwdTcParams::CTAS_PER_SM)
    bed_backward_tc_kernel(const float* __restrict__ V, const float* __restrict__ lam,
                           const float* __restrict__ gV, const float* __restrict__ gL,
                           float* __restrict__ gA, int64_t batch, int n, int degree,
                           int32_t* __restrict__ status_out, int32_t* __restrict__ flags) {
  using P = BwdTcParams;
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  uint8_t* const smem = tc_smem;
  auto buf = [&](int op, int part) { return smem + (2 * op + part) * P::BUF; };
  float* sLam = reinterpret_cast<float*>(smem + P::OFF_LAM);
  float* sInv = sLam + 64;
  float* sGl = sInv + 64;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + P::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + P::OFF_TMEM);
  int* outside = reinterpret_cast<int*>(smem + P::OFF_OUT);
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
  // epilogue geometry (M = 64): row m of D sits in TMEM lane 32 (m / 16) +
  // m % 16, so warp w reads its subpartition's lanes (w % 4) and keeps lanes
  // 0-15; warps w and w + 4 split the 64 columns
  const int sub = warp & 3, ch = warp >> 2;
  const int r = 16 * sub + (lane & 15);  // row of D this thread holds
  const int c_lo = 32 * ch;
  const int c_half = lane < 16 ? 0 : 8;  // split_half: this lane's 8 of each 16 columns
  const uint32_t trow = tmem + ((uint32_t)(32 * sub) << 16) + (uint32_t)c_lo;

  // D = A B^T over K = 64 (3xTF32)
  auto issue = [&](int opA, int opB) {
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_hi = smem_u32(buf(opA, 0)), a_lo = smem_u32(buf(opA, 1));
      const uint32_t b_hi = smem_u32(buf(opB, 0)), b_lo = smem_u32(buf(opB, 1));
      constexpr uint32_t lbo = 128u, sbo = 2048u, step = 256u;
      constexpr uint32_t idesc = kIdescTf32;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t o = step * kk;
        umma_tf32(tmem, umma_desc(a_lo + o, lbo, sbo), umma_desc(b_hi + o, lbo, sbo), idesc, kk > 0 ? 1u : 0u);
        umma_tf32(tmem, umma_desc(a_hi + o, lbo, sbo), umma_desc(b_lo + o, lbo, sbo), idesc, 1u);
        umma_tf32(tmem, umma_desc(a_hi + o, lbo, sbo), umma_desc(b_hi + o, lbo, sbo), idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(bar))
                   : "memory");
    }
  };
  auto wait_mma = [&]() {
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
  };
  auto sync_for_mma = [&]() {  // generic-proxy smem writes -> the tensor core
    proxy_fence_smem();
    tc_fence_before();
    __syncthreads();
  };

  // ---- stage: X1 = gV^T, X2 = V^T, X3 = V (zero padded to 64), hi/lo.  A
  // warp covers one 8-row x 4-k core block per step: lane -> (row 8rb +
  // lane/4, k 4kb + lane%4), so the 32 lanes hit 32 distinct banks.  The next
  // matrix's loads are issued while this one's last product runs (prefetch),
  // its stores at the top of the next iteration (stage).
  constexpr int kStageU = 16;  // 128 core blocks / 8 warps
  float p_kr[kStageU], p_g[kStageU], p_l = 0.0f, p_gl = 0.0f;
  auto prefetch = [&](int64_t mm) {
    const bool have = mm < batch;
    const float* vb = V + (have ? mm : 0) * nn;
    const float* gb = gV ? gV + (have ? mm : 0) * nn : nullptr;
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int c = warp + 8 * u;
      const int row = 8 * (c >> 4) + (lane >> 2), k = 4 * (c & 15) + (lane & 3);
      const bool ok = have && row < n && k < n;
      p_kr[u] = ok ? __ldg(vb + k * n + row) : 0.0f;  // V[k][row]
      p_g[u] = (ok && gb) ? __ldg(gb + k * n + row) : 0.0f;
    }
    const bool okl = have && tid < n;
    p_l = okl ? __ldg(lam + mm * n + tid) : 0.0f;
    p_gl = (okl && gL) ? __ldg(gL + mm * n + tid) : 0.0f;
  };
  const bool vec4 = (n % 4 == 0) && (reinterpret_cast<uintptr_t>(V) & 15) == 0;
  prefetch(blockIdx.x);
  for (int64_t m = blockIdx.x; m < batch; m += gridDim.x) {
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int c = warp + 8 * u;
      const uint32_t o = kmaj_off(8 * (c >> 4) + (lane >> 2), 4 * (c & 15) + (lane & 3));
      float x;
      x = tf32_hi(p_g[u]);
      *reinterpret_cast<float*>(buf(0, 0) + o) = x;
      *reinterpret_cast<float*>(buf(0, 1) + o) = tf32_hi(p_g[u] - x);
      x = tf32_hi(p_kr[u]);
      *reinterpret_cast<float*>(buf(1, 0) + o) = x;
      *reinterpret_cast<float*>(buf(1, 1) + o) = tf32_hi(p_kr[u] - x);
    }
    bool pos = true;
    if (tid < 64) {
      const float l = p_l;
      sLam[tid] = l;
      sInv[tid] = l != 0.0f ? 1.0f / l : 0.0f;
      sGl[tid] = p_gl;
      pos = tid >= n || l > 0.0f;
      if (tid == 0) outside[0] = 0;
    }
    proxy_fence_smem();
    tc_fence_before();
    // every eigenvalue positive: F needs no domain checks
    const bool all_pos = __syncthreads_and(pos) != 0;

    // ---- P1: D = gV^T V = M^T;  E1: M'^T[r][c] = F(c, r) M[c][r] + (c == r) gL[r] -> X1
    issue(0, 1);
    // V as stored (the A of P2, the B of P3) goes into X2 once P1 has read V^T
    // from it: its 128-bit loads are issued now, the stores after E1
    float4 vr[4];
    {
      const float* vb = V + m * nn;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = warp + 8 * u;  // 32 core-block steps: 8 rows x 4 k-groups each
        const int row = 8 * (c >> 2) + (lane & 7), k0 = 4 * (4 * (c & 3) + (lane >> 3));
        vr[u] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (row < n && k0 < n) {
          const float* src = vb + row * n + k0;
          if (vec4) {
            vr[u] = __ldg(reinterpret_cast<const float4*>(src));
          } else {
            vr[u].x = __ldg(src);
            vr[u].y = k0 + 1 < n ? __ldg(src + 1) : 0.0f;
            vr[u].z = k0 + 2 < n ? __ldg(src + 2) : 0.0f;
            vr[u].w = k0 + 3 < n ? __ldg(src + 3) : 0.0f;
          }
        }
      }
    }
    wait_mma();
    {
      bool off = false;
      const float lr = sLam[r], ir = sInv[r];
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const int cb = c_lo + 16 * q + c_half;
        float d[16], e[8];
        tmem_ld16(trow + 16u * q, d);
        tmem_wait_ld();
        split_half(d, lane, e);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = cb + j;
          const float lc = sLam[c], icv = sInv[c];
          const float f = all_pos ? taylor_f<false>(c, r, lc, lr, icv, ir, degree, n, off)
                                  : taylor_f<true>(c, r, lc, lr, icv, ir, degree, n, off);
          e[j] = f * e[j] + (c == r ? sGl[r] : 0.0f);
        }
        store8(buf(0, 0), buf(0, 1), r, cb, e);
      }
      if (off) atomicOr(&outside[0], 1);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = warp + 8 * u;
      const int row = 8 * (c >> 2) + (lane & 7), k0 = 4 * (4 * (c & 3) + (lane >> 3));
      const float4 v = vr[u];
      const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
      const uint32_t o = kmaj_off(row, k0);
      *reinterpret_cast<float4*>(buf(1, 0) + o) = h;
      *reinterpret_cast<float4*>(buf(1, 1) + o) =
          make_float4(tf32_hi(v.x - h.x), tf32_hi(v.y - h.y), tf32_hi(v.z - h.z), tf32_hi(v.w - h.w));
    }
    sync_for_mma();
    // ---- P2: D = V M' = W;  E2: W -> X1 (A of P3; P2 has read M'^T)
    issue(1, 0);
    wait_mma();
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      float d[16], e[8];
      tmem_ld16(trow + 16u * q, d);
      tmem_wait_ld();
      split_half(d, lane, e);
      store8(buf(0, 0), buf(0, 1), r, c_lo + 16 * q + c_half, e);
    }
    sync_for_mma();
    // ---- P3: D = W V^T = G;  E3: G through the X1 region (P3 has read W)
    issue(0, 1);
    prefetch(m + gridDim.x);  // in flight during P3, E3 and the stores
    wait_mma();
    float* sg = reinterpret_cast<float*>(buf(0, 0));
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
    if (tid == 0) {
      const int st = outside[0] ? kStatusNonPositive : kStatusOk;
      if (status_out) status_out[m] = st;
      if (flags && st) atomicOr(flags, 1 << st);
    }
    // gA = (G + G^T) / 2, one row per warp step, coalesced along columns
    for (int rr = warp; rr < n; rr += P::THREADS / 32) {
      float* dst = gA + m * nn + rr * n;
      const float* grow = sg + rr * P::SPITCH;
      const float* gcol = sg + rr;
      dst[lane] = 0.5f * (grow[lane] + gcol[lane * P::SPITCH]);  // n > 32: lanes 0..31 all valid
      if (lane + 32 < n) dst[lane + 32] = 0.5f * (grow[lane + 32] + gcol[(lane + 32) * P::SPITCH]);
    }
    __syncthreads();  // the stage (X1) is rewritten by the next matrix
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

}  // namespace bed

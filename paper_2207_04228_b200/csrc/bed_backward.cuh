// bed_backward.cuh -- ED backward with the Taylor-polynomial K.
//
//   gA = sym( V (F o (V^T gV) + diag(gL)) V^T ),  sym(M) = (M + M^T)/2
//   F_ij ~ 1/(l_j - l_i):  for the pair's larger value l_big (index order on
//   ties) and smaller l_small,  T = (1/l_big) sum_{k=0..K} (l_small/l_big)^k,
//   F_ij = -T when l_i is the larger, +T otherwise; F_ii = 0.
// The series converges to 1/(l_j - l_i) only for |l_small / l_big| < 1 (and
// equals (K+1)/l on ties), i.e. on the positive spectra of the paper's
// covariance inputs.  A pair outside that domain
// (l_big <= 0, or l_small <= -l_big) takes the exact 1/(l_j - l_i) instead
// and its matrix is reported as BED_STATUS_NON_POSITIVE (a pair of zeros,
// or a tie outside the domain, gives F = 0).
//
// The reference package has no backward (pkg/README.md:116-117); the paper
// reuses [song2021approximate] with a degree-9 Taylor polynomial
// (PAPER.md:668, :700).  The float64 restatement checked against this
// kernel is oracle/oracle.py:taylor_backward.
//
// Three n x n x n products per matrix, FP32 on the FMA pipe (no tensor
// cores: the gradient gate is 1e-4 relative, beyond TF32):
//   M = V^T gV      (then M' = F o M + diag(gL), F built in the epilogue)
//   W = V M'
//   G = W V^T       (gA = (G + G^T) / 2 through the shared stage)
// Each thread owns a 4 x 4 output tile; per k it reads a 4-wide column slice
// of A and a 4-wide row slice of B as two 128-bit shared loads and issues 8
// FFMA2 (16 FMAs), so the products run at the FMA-pipe rate.  Every operand
// is kept in the orientation its product reads: V, V^T, and the
// intermediate results written transposed where the next product needs it.
#pragma once

#include "bed_common.cuh"
#include "bed_f32x2.cuh"
#include "bed_tile.cuh"

namespace bed {

template <int NMAX>
struct BwdParams {
  static constexpr int TQ = NMAX / 4;                 // tiles per row
  static constexpr int TPM = TQ * TQ;                  // threads per matrix
  static constexpr int MB = TPM >= 128 ? 1 : 128 / TPM;  // matrices per CTA
  static constexpr int THREADS = MB * TPM;
  static constexpr int SROW = NMAX + 4;                // 16-byte rows
  static constexpr int SBUF = NMAX * SROW;
  static constexpr int PER = 3 * SBUF + 2 * NMAX;      // V, V^T, X (gV -> M' -> G), lam, 1/lam
  static constexpr size_t BYTES = sizeof(float) * (size_t)MB * PER;
};

// acc (4 x 4 tile as [row][col pair]) += A(rows, k) B(k, cols) over k, with
// At the k-major copy of A (At + k*SROW + r is A(r, k)) and B row-major.
template <int NMAX, int SROW>
__device__ __forceinline__ void tile_gemm(const float* At, const float* B, int ti, int tj,
                                          f2 (&acc)[4][2]) {
#pragma unroll
  for (int k = 0; k < NMAX; ++k) {
    const float4 a = *reinterpret_cast<const float4*>(At + k * SROW + 4 * ti);
    const float4 b = *reinterpret_cast<const float4*>(B + k * SROW + 4 * tj);
    const f2 b0 = f2_make(b.x, b.y), b1 = f2_make(b.z, b.w);
    acc[0][0] = ffma2(f2_bc(a.x), b0, acc[0][0]);
    acc[0][1] = ffma2(f2_bc(a.x), b1, acc[0][1]);
    acc[1][0] = ffma2(f2_bc(a.y), b0, acc[1][0]);
    acc[1][1] = ffma2(f2_bc(a.y), b1, acc[1][1]);
    acc[2][0] = ffma2(f2_bc(a.z), b0, acc[2][0]);
    acc[2][1] = ffma2(f2_bc(a.z), b1, acc[2][1]);
    acc[3][0] = ffma2(f2_bc(a.w), b0, acc[3][0]);
    acc[3][1] = ffma2(f2_bc(a.w), b1, acc[3][1]);
  }
}

__device__ __forceinline__ float tile_at(const f2 (&acc)[4][2], int i, int j) {
  return (j & 1) ? f2_hi(acc[i][j >> 1]) : f2_lo(acc[i][j >> 1]);
}

template <int NMAX, bool EXACT>
__global__ void __launch_bounds__(BwdParams<NMAX>::THREADS)
    bed_backward_kernel(const float* __restrict__ V, const float* __restrict__ lam,
                        const float* __restrict__ gV, const float* __restrict__ gL,
                        float* __restrict__ gA, int64_t batch, int n_rt, int degree,
                        int32_t* __restrict__ status_out, int32_t* __restrict__ flags) {
  using P = BwdParams<NMAX>;
  constexpr int SROW = P::SROW, TQ = P::TQ;
  const int n = EXACT ? NMAX : n_rt;
  const int nn = n * n;
  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int mi = tid / P::TPM;
  const int t = tid % P::TPM;
  const int ti = t / TQ, tj = t % TQ;
  const int64_t base = (int64_t)blockIdx.x * P::MB;
  const int count = (batch - base) < P::MB ? (int)(batch - base) : P::MB;
  float* sV = smem + mi * P::PER;  // V, row-major
  float* sT = sV + P::SBUF;        // V^T, later read as the B of G = W V^T
  float* sX = sT + P::SBUF;        // gV -> M' -> G
  float* sL = sX + P::SBUF;
  float* sI = sL + NMAX;
  __shared__ int outside[P::MB];  // matrix has a pair outside the Taylor domain

  if (!EXACT) {  // padding rows/columns must read as zeros in the products
    for (int g = tid; g < P::MB * P::PER; g += P::THREADS) smem[g] = 0.0f;
    __syncthreads();
  }
  // ---- coalesced loads of V and gV into the stage, eigenvalues
  // (the generic copy targets one buffer per matrix at stride PER)
  // V and gV: every 16-byte word in flight at once (cp.async) when the tile allows
  const bool av = tile_to_stage_async<NMAX, P::THREADS, SROW, P::PER>(V + base * nn, count, n, smem);
  const bool ag = gV ? tile_to_stage_async<NMAX, P::THREADS, SROW, P::PER>(gV + base * nn, count, n,
                                                                           smem + 2 * P::SBUF)
                     : true;
  cp_async_commit();
  if (!av) tile_to_stage<NMAX, P::THREADS, SROW, P::PER>(V + base * nn, count, n, smem);
  if (!ag) tile_to_stage<NMAX, P::THREADS, SROW, P::PER>(gV + base * nn, count, n, smem + 2 * P::SBUF);
  for (int g = tid; g < count * n; g += P::THREADS) {
    const int mat = g / n, c = g - mat * n;
    const float l = __ldg(lam + base * n + g);
    float* dl = smem + mat * P::PER + 3 * P::SBUF;
    dl[c] = l;
    dl[NMAX + c] = l != 0.0f ? 1.0f / l : 0.0f;
  }
  cp_async_wait_all();
  __syncthreads();
  for (int g = tid; g < P::MB; g += P::THREADS) outside[g] = 0;
  // V^T from V
  for (int g = tid; g < P::MB * NMAX * NMAX; g += P::THREADS) {
    const int mat = g / (NMAX * NMAX), off = g - mat * NMAX * NMAX;
    const int r = off / NMAX, c = off - r * NMAX;
    float* b = smem + mat * P::PER;
    b[P::SBUF + c * SROW + r] = b[r * SROW + c];
  }
  __syncthreads();

  const bool live = mi < count;
  f2 acc[4][2];
  // The three products share one copy of the tile GEMM (a runtime loop keeps
  // the kernel's code inside the instruction cache):
  //   ph 0: M = V^T gV, then M' = F o M + diag(gL) in the epilogue
  //   ph 1: W = V M' (A = V, read k-major from V^T); W^T goes to sV
  //   ph 2: G = W V^T (A = W, k-major from W^T; B(j, c) = V(c, j) = V^T row j)
#pragma unroll 1
  for (int ph = 0; ph < 3; ++ph) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = f2_bc(0.0f);
    if (ph > 0 || gV) tile_gemm<NMAX, SROW>(ph == 1 ? sT : sV, ph == 2 ? sT : sX, ti, tj, acc);
    if (ph == 0) {
      // F by Horner in packed pairs (two tile columns per FFMA2)
      float mp[4][4];
      bool off_domain = false;
      // a tile whose eight eigenvalues are all positive is inside the series'
      // domain (0 < l_small <= l_big): no per-pair check
      float tmin = sL[4 * ti];
    #pragma unroll
      for (int q = 0; q < 4; ++q) tmin = fminf(tmin, fminf(sL[4 * ti + q], sL[4 * tj + q]));
      const bool tile_pos = tmin > 0.0f;
    #pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int i = 4 * ti + ii;
        const float li = sL[i], ii_inv = sI[i];
        const float gli = (gL && i < n && ti == tj && live) ? __ldg(gL + (base + mi) * n + i) : 0.0f;
    #pragma unroll
        for (int jp = 0; jp < 2; ++jp) {
          float ratio[2], binv[2];
          bool hf[2];
    #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 4 * tj + 2 * jp + h;
            const float lj = sL[j];
            hf[h] = i < j ? (li >= lj) : (li > lj);
            binv[h] = hf[h] ? ii_inv : sI[j];
            ratio[h] = (hf[h] ? lj : li) * binv[h];
          }
          const f2 rt = f2_make(ratio[0], ratio[1]);
          f2 poly = f2_bc(1.0f);
          for (int k = 0; k < degree; ++k) poly = ffma2(poly, rt, f2_bc(1.0f));
          const f2 tt = fmul2(poly, f2_make(binv[0], binv[1]));
    #pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int jj = 2 * jp + h, j = 4 * tj + jj;
            float tv = h ? f2_hi(tt) : f2_lo(tt);
            if (!tile_pos) {
              // the series' domain: l_big > 0 and |ratio| < 1, or a tie (ratio 1)
              const float lj = sL[j];
              const float big = hf[h] ? li : lj, small = hf[h] ? lj : li;
              const bool in_domain = (big > 0.0f && (fabsf(ratio[h]) < 1.0f || small == big)) ||
                                     (big == 0.0f && small == 0.0f);
              if (!in_domain && i != j && i < n && j < n) {
                tv = big != small ? 1.0f / (big - small) : 0.0f;  // exact 1/(l_j - l_i), sign below
                off_domain = true;
              }
            }
            const float f = i == j ? 0.0f : (hf[h] ? -tv : tv);
            mp[ii][jj] = f * tile_at(acc, ii, jj) + (i == j ? gli : 0.0f);
          }
        }
      }
      if (off_domain && live) atomicOr(&outside[mi], 1);
      __syncthreads();  // every thread is done reading gV
      if (t == 0 && live) {
        const int st = outside[mi] ? kStatusNonPositive : kStatusOk;
        if (status_out) status_out[base + mi] = st;
        if (flags && st) atomicOr(flags, 1 << st);
      }
      if (live) {
    #pragma unroll
        for (int ii = 0; ii < 4; ++ii)
          *reinterpret_cast<float4*>(sX + (4 * ti + ii) * SROW + 4 * tj) =
              make_float4(mp[ii][0], mp[ii][1], mp[ii][2], mp[ii][3]);
      }
      __syncthreads();

    } else if (ph == 1) {
      if (live) {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
          *reinterpret_cast<float4*>(sV + (4 * tj + jj) * SROW + 4 * ti) =
              make_float4(tile_at(acc, 0, jj), tile_at(acc, 1, jj), tile_at(acc, 2, jj), tile_at(acc, 3, jj));
      }
      __syncthreads();
    } else {
      if (live) {  // sX (M') was last read by the W product, before the barrier
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
          *reinterpret_cast<float4*>(sX + (4 * ti + ii) * SROW + 4 * tj) =
              make_float4(tile_at(acc, ii, 0), tile_at(acc, ii, 1), tile_at(acc, ii, 2), tile_at(acc, ii, 3));
      }
      __syncthreads();
    }
  }
  // ---- gA = (G + G^T) / 2, coalesced
  for (int g = tid; g < count * nn; g += P::THREADS) {
    const int mat = g / nn, off = g - mat * nn;
    const int r = off / n, c = off - r * n;
    const float* gs = smem + mat * P::PER + 2 * P::SBUF;
    gA[base * nn + g] = 0.5f * (gs[r * SROW + c] + gs[c * SROW + r]);
  }
}

}  // namespace bed

// bed_backward.cuh -- ED backward with the Taylor-polynomial K.
//
//   gA = sym( V (F o (V^T gV) + diag(gL)) V^T ),  sym(M) = (M + M^T)/2
//   F_ij ~ 1/(l_j - l_i):  for the pair's larger value l_big (index order on
//   ties) and smaller l_small,  T = (1/l_big) sum_{k=0..K} (l_small/l_big)^k,
//   F_ij = -T when l_i is the larger, +T otherwise; F_ii = 0.
//
// The reference package has no backward (pkg/README.md:116-117); the paper
// reuses [song2021approximate] with a degree-9 Taylor polynomial
// (PAPER.md:668, :700).  The float64 restatement checked against this
// kernel is oracle/oracle.py:taylor_backward.
//
// Layout: NMAX threads per matrix, thread i owns row i of every n x n
// product; MB matrices per CTA.  Three n^3 FFMA products, all operands
// staged in shared memory with 16-byte-aligned rows so the broadcast
// operand reads are LDS.128; the final symmetrisation reads the transpose
// through an odd stride (conflict free); loads and stores are coalesced.
#pragma once

#include "bed_common.cuh"

namespace bed {

template <int NMAX>
struct BwdParams {
  static constexpr int MB = NMAX >= 64 ? 2 : 256 / NMAX;
  static constexpr int THREADS = MB * NMAX;
  static constexpr int SA = NMAX + 4;  // aligned stride (broadcast / row reads)
  static constexpr int SG = NMAX + 1;  // odd stride (transposed reads)
  static constexpr int PER = 2 * NMAX * SA + 2 * NMAX;  // V, X stages + lam, inv
  static constexpr size_t BYTES = sizeof(float) * (size_t)MB * PER;
};

template <int NMAX, bool EXACT>
__global__ void __launch_bounds__(BwdParams<NMAX>::THREADS)
    bed_backward_kernel(const float* __restrict__ V, const float* __restrict__ lam,
                        const float* __restrict__ gV, const float* __restrict__ gL,
                        float* __restrict__ gA, int64_t batch, int n_rt, int degree) {
  using P = BwdParams<NMAX>;
  constexpr int SA = P::SA, SG = P::SG;
  const int n = EXACT ? NMAX : n_rt;
  const int nn = n * n;
  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int mi = tid / NMAX;
  const int row = tid % NMAX;
  const int64_t base = (int64_t)blockIdx.x * P::MB;
  const int count = (batch - base) < P::MB ? (int)(batch - base) : P::MB;
  float* sV = smem + mi * P::PER;
  float* sX = sV + NMAX * SA;
  float* sL = sX + NMAX * SA;
  float* sI = sL + NMAX;

  if (!EXACT) {  // padding rows/columns must read as zeros in the products
    for (int g = tid; g < P::MB * P::PER; g += P::THREADS) smem[g] = 0.0f;
    __syncthreads();
  }
  // ---- coalesced loads of V and gV, plus the eigenvalues
  for (int g = tid; g < count * nn; g += P::THREADS) {
    int mat = g / nn, off = g - mat * nn;
    int r = off / n, c = off - r * n;
    float* dv = smem + mat * P::PER;
    dv[r * SA + c] = __ldg(V + base * nn + g);
    dv[NMAX * SA + r * SA + c] = gV ? __ldg(gV + base * nn + g) : 0.0f;
  }
  for (int g = tid; g < count * n; g += P::THREADS) {
    int mat = g / n, c = g - mat * n;
    float l = __ldg(lam + base * n + g);
    float* dl = smem + mat * P::PER + 2 * NMAX * SA;
    dl[c] = l;
    dl[NMAX + c] = l != 0.0f ? 1.0f / l : 0.0f;
  }
  __syncthreads();

  const bool live = mi < count && row < n;
  // ---- M(row, :) = sum_r V(r, row) gV(r, :)
  float acc[NMAX];
#pragma unroll
  for (int c = 0; c < NMAX; ++c) acc[c] = 0.0f;
  if (gV && live) {
    for (int r = 0; r < n; ++r) {
      const float vr = sV[r * SA + row];
      const float4* x4 = reinterpret_cast<const float4*>(sX + r * SA);
#pragma unroll
      for (int c4 = 0; c4 < NMAX / 4; ++c4) {
        float4 x = x4[c4];
        acc[4 * c4 + 0] = fmaf(vr, x.x, acc[4 * c4 + 0]);
        acc[4 * c4 + 1] = fmaf(vr, x.y, acc[4 * c4 + 1]);
        acc[4 * c4 + 2] = fmaf(vr, x.z, acc[4 * c4 + 2]);
        acc[4 * c4 + 3] = fmaf(vr, x.w, acc[4 * c4 + 3]);
      }
    }
  }
  // ---- M' = F o M + diag(gL)
  if (live) {
    const float li = sL[row];
#pragma unroll
    for (int c = 0; c < NMAX; ++c) {
      if (c < n) {
        float f = 0.0f;
        if (c != row) {
          const float lc = sL[c];
          const bool hi_first = row < c ? (li >= lc) : (li > lc);
          const float big_inv = hi_first ? sI[row] : sI[c];
          const float small = hi_first ? lc : li;
          const float ratio = small * big_inv;
          float poly = 1.0f;
          for (int k = 0; k < degree; ++k) poly = fmaf(poly, ratio, 1.0f);
          const float t = big_inv * poly;
          f = hi_first ? -t : t;
        }
        acc[c] *= f;
      } else {
        acc[c] = 0.0f;
      }
    }
  }
  __syncthreads();  // every thread is done reading gV
  if (mi < count) {
    float* xr = sX + row * SA;
#pragma unroll
    for (int c = 0; c < NMAX; ++c) xr[c] = live ? acc[c] : 0.0f;
    if (live && gL) xr[row] += __ldg(gL + (base + mi) * n + row);
  }
  __syncthreads();

  // ---- W(row, :) = V(row, :) M'
  float vrow[NMAX];
#pragma unroll
  for (int c = 0; c < NMAX; ++c) {
    vrow[c] = live ? sV[row * SA + c] : 0.0f;
    acc[c] = 0.0f;
  }
#pragma unroll
  for (int i = 0; i < NMAX; ++i) {
    if (!EXACT && i >= n) break;
    const float vi = vrow[i];
    const float4* x4 = reinterpret_cast<const float4*>(sX + i * SA);
#pragma unroll
    for (int c4 = 0; c4 < NMAX / 4; ++c4) {
      float4 x = x4[c4];
      acc[4 * c4 + 0] = fmaf(vi, x.x, acc[4 * c4 + 0]);
      acc[4 * c4 + 1] = fmaf(vi, x.y, acc[4 * c4 + 1]);
      acc[4 * c4 + 2] = fmaf(vi, x.z, acc[4 * c4 + 2]);
      acc[4 * c4 + 3] = fmaf(vi, x.w, acc[4 * c4 + 3]);
    }
  }
  // ---- G(row, c) = sum_i W(row, i) V(c, i)
  float gr[NMAX];
#pragma unroll
  for (int c = 0; c < NMAX; ++c) {
    float s = 0.0f;
    if (EXACT || c < n) {
      const float4* v4 = reinterpret_cast<const float4*>(sV + c * SA);
#pragma unroll
      for (int i4 = 0; i4 < NMAX / 4; ++i4) {
        float4 x = v4[i4];
        s = fmaf(acc[4 * i4 + 0], x.x, s);
        s = fmaf(acc[4 * i4 + 1], x.y, s);
        s = fmaf(acc[4 * i4 + 2], x.z, s);
        s = fmaf(acc[4 * i4 + 3], x.w, s);
      }
    }
    gr[c] = s;
  }
  __syncthreads();  // done reading M' from sX
  if (mi < count) {
    float* gout = sX + row * SG;
#pragma unroll
    for (int c = 0; c < NMAX; ++c) gout[c] = gr[c];
  }
  __syncthreads();
  for (int g = tid; g < count * nn; g += P::THREADS) {
    int mat = g / nn, off = g - mat * nn;
    int r = off / n, c = off - r * n;
    const float* gs = smem + mat * P::PER + NMAX * SA;
    gA[base * nn + g] = 0.5f * (gs[r * SG + c] + gs[c * SG + r]);
  }
}

}  // namespace bed

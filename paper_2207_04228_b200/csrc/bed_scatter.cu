// bed_scatter.cu -- the covariance producer in front of the ED (SURVEY.md
// 8(f) row 3): out = (X - mu)(X - mu)^T + eps I per matrix, X (batch, n, m)
// row-major (n channels, m samples), mu the per-channel sample mean -- the
// scatter of the reference zca_whiten (solver.py:161-166) and of
// decorrelated BN / global covariance pooling.
//
// n <= 8 takes the one-thread-per-matrix producer of bed_scatter_regs.cuh.
// Above, a CTA owns 128 / (NMAX/4)^2 matrices (one for n > 32): pass 1 reduces the channel means
// (one warp per channel row, coalesced), pass 2 streams the centred
// samples in chunks of KC through shared memory k-major (X_c^T) and
// accumulates X_c X_c^T on the 4 x 4 FFMA2 register tiles of the backward
// (both operands are the same k-major chunk).  The result is symmetrised
// through the stage like the reference ((S + S^T) / 2, solver.py:164).
#include "bed_backward.cuh"
#include "bed_launch.h"
#include "bed_scatter_regs.cuh"
#include "bed_scatter_tc.cuh"

#include <stdlib.h>

namespace bed {

template <int NMAX>
struct ScatParams {
  static constexpr int TQ = NMAX / 4;
  static constexpr int TPM = TQ * TQ;                   // tile owners per matrix
  static constexpr int MB = TPM >= 128 ? 1 : 128 / TPM;  // matrices per CTA
  static constexpr int THREADS = MB * TPM;
  static constexpr int KC = 32;                         // samples per staged chunk
  static constexpr int ROWS = MB * NMAX;                // (matrix, channel) row-sum owners
  static constexpr int RPT = (ROWS + THREADS - 1) / THREADS;  // owners per thread
  static constexpr int SROW = NMAX + 4;
  static constexpr int PER = KC * SROW + NMAX + NMAX * (NMAX + 1);  // X_c^T chunk, mu, result
  static constexpr size_t BYTES = sizeof(float) * (size_t)MB * PER;
};

template <int NMAX>
__device__ __forceinline__ void tile_gemm_chunk(const float* XT, int ti, int tj, int kc, f2 (&acc)[4][2]) {
  constexpr int SROW = ScatParams<NMAX>::SROW;
#pragma unroll 8
  for (int k = 0; k < kc; ++k) {
    const float4 a = *reinterpret_cast<const float4*>(XT + k * SROW + 4 * ti);
    const float4 b = *reinterpret_cast<const float4*>(XT + k * SROW + 4 * tj);
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

template <int NMAX>
__global__ void __launch_bounds__(ScatParams<NMAX>::THREADS)
    bed_scatter_kernel(const float* __restrict__ X, float* __restrict__ out, int64_t batch, int n,
                       int m, float eps) {
  using P = ScatParams<NMAX>;
  constexpr int SROW = P::SROW, TQ = P::TQ, KC = P::KC;
  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = P::THREADS / 32;
  const int64_t base = (int64_t)blockIdx.x * P::MB;
  const int count = (batch - base) < P::MB ? (int)(batch - base) : P::MB;
  const float* x = X + base * n * m;
  auto buf = [&](int mat) { return smem + mat * P::PER; };

  // One pass over X, shifted by each channel's first sample x0 (which keeps
  // the one-pass formula free of cancellation at the data's spread, not its
  // offset):  S = sum_k (x_k - x0)(x_k - x0)^T - m d d^T,  d = mean(x - x0).
  // The shift goes in the mean slot; the k-major chunks feed the 4 x 4
  // FFMA2 tiles, and one thread per channel row sums its chunk column.
  for (int g = tid; g < P::MB * NMAX; g += P::THREADS) {
    const int mat = g / NMAX, r = g - mat * NMAX;
    buf(mat)[KC * SROW + r] = (mat < count && r < n) ? __ldg(x + ((int64_t)mat * n + r) * m) : 0.0f;
  }
  __syncthreads();
  (void)lane;
  (void)warp;
  (void)NWARP;
  const int mi = tid / P::TPM, t = tid % P::TPM;
  const int ti = t / TQ, tj = t % TQ;
  // Row-sum owners: (matrix, channel) pairs o = tid + q * THREADS, strided
  // so every pair of the CTA has one (ROWS can exceed THREADS for n <= 8).
  float rowsum[P::RPT];
#pragma unroll
  for (int q = 0; q < P::RPT; ++q) rowsum[q] = 0.0f;
  f2 acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = f2_bc(0.0f);
  for (int k0 = 0; k0 < m; k0 += KC) {
    const int kc = min(KC, m - k0);
#pragma unroll 4
    for (int g = tid; g < P::MB * NMAX * KC; g += P::THREADS) {  // coalesced along samples
      const int rr = g / KC, k = g - rr * KC;
      const int mat = rr / NMAX, r = rr - mat * NMAX;
      float v = 0.0f;
      if (mat < count && r < n && k < kc)
        v = __ldg(x + ((int64_t)mat * n + r) * m + k0 + k) - buf(mat)[KC * SROW + r];
      buf(mat)[k * SROW + r] = v;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < P::RPT; ++q) {
      const int o = tid + q * P::THREADS;
      if (o < P::ROWS) {
        const float* col = buf(o / NMAX) + o % NMAX;
        for (int k = 0; k < kc; ++k) rowsum[q] += col[k * SROW];
      }
    }
    tile_gemm_chunk<NMAX>(buf(mi), ti, tj, kc, acc);
    __syncthreads();
  }
  // d = rowsum / m into the stage row the chunks used (no longer needed)
#pragma unroll
  for (int q = 0; q < P::RPT; ++q) {
    const int o = tid + q * P::THREADS;
    if (o < P::ROWS) buf(o / NMAX)[o % NMAX] = rowsum[q] / (float)m;
  }
  __syncthreads();
  {
    const float* dv = buf(mi);
    const float fm = (float)m;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const float di = dv[4 * ti + ii] * fm;
#pragma unroll
      for (int jp = 0; jp < 2; ++jp)
        acc[ii][jp] = ffma2(f2_bc(-di), f2_make(dv[4 * tj + 2 * jp], dv[4 * tj + 2 * jp + 1]), acc[ii][jp]);
    }
  }
  float* cs = buf(mi) + KC * SROW + NMAX;
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) cs[(4 * ti + ii) * (NMAX + 1) + 4 * tj + jj] = tile_at(acc, ii, jj);
  __syncthreads();
  const int nn = n * n;
  for (int g = tid; g < count * nn; g += P::THREADS) {
    const int mat = g / nn, off = g - mat * nn;
    const int r = off / n, c = off - r * n;
    const float* c2 = buf(mat) + KC * SROW + NMAX;
    float v = 0.5f * (c2[r * (NMAX + 1) + c] + c2[c * (NMAX + 1) + r]);
    if (r == c) v += eps;
    out[base * nn + g] = v;
  }
}

template <int NMAX>
static cudaError_t go_scatter(const ScatArgs& a) {
  using P = ScatParams<NMAX>;
  auto kern = bed_scatter_kernel<NMAX>;
  if (cudaError_t e = ensure_smem(kern, P::BYTES); e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.batch + P::MB - 1) / P::MB);
  kern<<<grid, P::THREADS, P::BYTES, a.stream>>>(a.X, a.out, a.batch, a.n, a.m, a.eps);
  return cudaGetLastError();
}

template <int N>
static cudaError_t go_scatter_small(const ScatArgs& a) {
  const unsigned grid = (unsigned)((a.batch + kScatSmallThreads - 1) / kScatSmallThreads);
  bed_scatter_small_kernel<N><<<grid, kScatSmallThreads, 0, a.stream>>>(a.X, a.out, a.batch, a.m, a.eps);
  return cudaGetLastError();
}

// 33 <= n <= 64 on the tensor cores (bed_scatter_tc.cuh); BED_TC=0 selects
// the FFMA2 kernel
static bool scat_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("BED_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

static cudaError_t go_scatter_tc(const ScatArgs& a) {
  auto kern = bed_scatter_tc_kernel;
  if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), ScatTcParams::BYTES); e != cudaSuccess)
    return e;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t slots = (int64_t)ScatTcParams::CTAS_PER_SM * sms;
  const unsigned grid = (unsigned)(a.batch < slots ? a.batch : slots);
  kern<<<grid, ScatTcParams::THREADS, ScatTcParams::BYTES, a.stream>>>(a.X, a.out, a.batch, a.n, a.m, a.eps);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const ScatArgs& a) {
  if (a.n > 32 && scat_tc_enabled()) return go_scatter_tc(a);
  switch (a.n) {  // n <= 8: one thread per matrix (bed_scatter_regs.cuh)
    case 1: return go_scatter_small<1>(a);
    case 2: return go_scatter_small<2>(a);
    case 3: return go_scatter_small<3>(a);
    case 4: return go_scatter_small<4>(a);
    case 5: return go_scatter_small<5>(a);
    case 6: return go_scatter_small<6>(a);
    case 7: return go_scatter_small<7>(a);
    case 8: return go_scatter_small<8>(a);
    default: break;
  }
  if (a.n <= 16) return go_scatter<16>(a);
  if (a.n <= 32) return go_scatter<32>(a);
  return go_scatter<64>(a);
}

}  // namespace bed

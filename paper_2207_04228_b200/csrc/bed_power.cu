// bed_power.cu -- spectral power V diag(f(lambda)) V^T of a decomposed batch,
// f(l) = max(l, floor)^p: the reference matrix_power (solver.py:115-143),
// the consumer of the ED in decorrelated BN / ZCA whitening / global
// covariance pooling.
//
// One n x n x n product per matrix on the 4 x 4 FFMA2 register tiles of the
// backward (bed_backward.cuh): out(r, c) = sum_k V(r, k) f_k V(c, k), with
// A read k-major from V^T and B = diag(f) V^T, both staged in shared memory;
// the result is symmetrised through the stage like the reference
// ((out + out^T) / 2, solver.py:141).
//
// Floors (solver.py:127-132): floor < 0 selects the reference default
// 1e-12 * lambda_max per matrix; otherwise the absolute floor.  A negative
// or fractional p with a non-positive clamped eigenvalue flags the matrix
// (status 4 = NonPositiveSpectrum, solver.py:133-139) and writes zeros.
#include "bed_backward.cuh"
#include "bed_launch.h"
#include "bed_power_tc.cuh"

#include <stdlib.h>

namespace bed {

template <int NMAX>
struct PowParams {
  static constexpr int TQ = NMAX / 4;
  static constexpr int TPM = TQ * TQ;
  static constexpr int MB = TPM >= 128 ? 1 : 128 / TPM;
  static constexpr int THREADS = MB * TPM;
  static constexpr int SROW = NMAX + 4;
  static constexpr int SBUF = NMAX * SROW;
  static constexpr int PER = 3 * SBUF + NMAX;  // V (then C), V^T, diag(f) V^T, f
  static constexpr size_t BYTES = sizeof(float) * (size_t)MB * PER;
};

template <int NMAX, bool EXACT>
__global__ void __launch_bounds__(PowParams<NMAX>::THREADS)
    bed_power_kernel(const float* __restrict__ V, const float* __restrict__ lam,
                     float* __restrict__ out, int32_t* __restrict__ status,
                     int32_t* __restrict__ flags, int64_t batch, int n_rt, float p, float floor_abs,
                     int needs_positive, int merge) {
  using P = PowParams<NMAX>;
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
  float* sV = smem + mi * P::PER;
  float* sT = sV + P::SBUF;
  float* sF = sT + P::SBUF;
  float* sf = sF + P::SBUF;

  if (!EXACT) {
    for (int g = tid; g < P::MB * P::PER; g += P::THREADS) smem[g] = 0.0f;
    __syncthreads();
  }
  const bool vasync = tile_to_stage_async<NMAX, P::THREADS, SROW, P::PER>(V + base * nn, count, n, smem);
  cp_async_commit();
  if (!vasync) tile_to_stage<NMAX, P::THREADS, SROW, P::PER>(V + base * nn, count, n, smem);
  // f per eigenvalue; one thread per matrix resolves the floor and the
  // positivity check (n <= 64 values)
  if (t == 0 && mi < count) {
    const float* l = lam + (base + mi) * n;
    float lmax = -INFINITY;
    for (int c = 0; c < n; ++c) lmax = fmaxf(lmax, __ldg(l + c));
    const float fl = floor_abs < 0.0f ? 1e-12f * lmax : floor_abs;
    bool bad = false;
    for (int c = 0; c < n; ++c) {
      const float x = fmaxf(__ldg(l + c), fl);
      bad = bad || (needs_positive && !(x > 0.0f));
      sf[c] = x;
    }
    for (int c = 0; c < n; ++c) sf[c] = bad ? 0.0f : spectral_pow(sf[c], p);
    // merge (after a forward): a matrix the forward flagged keeps its status;
    // an accepted one is flagged only for a non-positive spectrum
    bool flag = bad;
    if (merge) flag = bad && (!status || status[base + mi] == kStatusOk);
    if (status && (flag || !merge)) status[base + mi] = flag ? kStatusNonPositive : kStatusOk;
    if (flag && flags) atomicOr(flags, 1 << kStatusNonPositive);
  }
  cp_async_wait_all();
  __syncthreads();
  // V^T and diag(f) V^T from V
  for (int g = tid; g < P::MB * NMAX * NMAX; g += P::THREADS) {
    const int mat = g / (NMAX * NMAX), off = g - mat * NMAX * NMAX;
    const int r = off / NMAX, c = off - r * NMAX;
    float* b = smem + mat * P::PER;
    const float x = b[r * SROW + c];
    b[P::SBUF + c * SROW + r] = x;
    b[2 * P::SBUF + c * SROW + r] = x * b[3 * P::SBUF + c];
  }
  __syncthreads();
  f2 acc[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = f2_bc(0.0f);
  tile_gemm<NMAX, SROW>(sT, sF, ti, tj, acc);
  if (mi < count) {  // sV is only read by the transposes above
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
      *reinterpret_cast<float4*>(sV + (4 * ti + ii) * SROW + 4 * tj) =
          make_float4(tile_at(acc, ii, 0), tile_at(acc, ii, 1), tile_at(acc, ii, 2), tile_at(acc, ii, 3));
  }
  __syncthreads();
  for (int g = tid; g < count * nn; g += P::THREADS) {
    const int mat = g / nn, off = g - mat * nn;
    const int r = off / n, c = off - r * n;
    const float* cs = smem + mat * P::PER;
    out[base * nn + g] = 0.5f * (cs[r * SROW + c] + cs[c * SROW + r]);
  }
}

template <int NMAX, bool EXACT>
static cudaError_t go_pow(const PowArgs& a) {
  using P = PowParams<NMAX>;
  auto kern = bed_power_kernel<NMAX, EXACT>;
  if (cudaError_t e = ensure_smem(kern, P::BYTES); e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.batch + P::MB - 1) / P::MB);
  kern<<<grid, P::THREADS, P::BYTES, a.stream>>>(a.V, a.lam, a.out, a.status, a.flags, a.batch,
                                                 a.n, a.p, a.floor_abs, a.needs_positive, a.merge);
  return cudaGetLastError();
}

template <int NMAX>
static cudaError_t go_pow_n(const PowArgs& a) {
  return a.n == NMAX ? go_pow<NMAX, true>(a) : go_pow<NMAX, false>(a);
}

// 33 <= n <= 64 on the tensor cores (bed_power_tc.cuh); BED_TC=0 selects the
// FFMA2 kernel
static bool pow_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("BED_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

static cudaError_t go_pow_tc(const PowArgs& a) {
  auto kern = bed_power_tc_kernel;
  if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), PowTcParams::BYTES); e != cudaSuccess)
    return e;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t slots = (int64_t)PowTcParams::CTAS_PER_SM * sms;
  const unsigned grid = (unsigned)(a.batch < slots ? a.batch : slots);
  kern<<<grid, PowTcParams::THREADS, PowTcParams::BYTES, a.stream>>>(
      a.V, a.lam, a.out, a.status, a.flags, a.batch, a.n, a.p, a.floor_abs, a.needs_positive, a.merge);
  return cudaGetLastError();
}

cudaError_t launch_power(const PowArgs& a) {
  if (a.n > 32 && pow_tc_enabled()) return go_pow_tc(a);
  if (a.n <= 4) return go_pow_n<4>(a);
  if (a.n <= 8) return go_pow_n<8>(a);
  if (a.n <= 16) return go_pow_n<16>(a);
  if (a.n <= 32) return go_pow_n<32>(a);
  return go_pow_n<64>(a);
}

}  // namespace bed

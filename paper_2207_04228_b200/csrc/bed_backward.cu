// Instantiations of the Taylor-K backward kernel.
#include "bed_backward.cuh"
#include "bed_backward_tc.cuh"
#include "bed_launch.h"

#include <stdlib.h>

namespace bed {

template <int NMAX, bool EXACT>
static cudaError_t go_bwd(const BwdArgs& a) {
  using P = BwdParams<NMAX>;
  auto kern = bed_backward_kernel<NMAX, EXACT>;
  if (cudaError_t e = ensure_smem(kern, P::BYTES); e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.batch + P::MB - 1) / P::MB);
  kern<<<grid, P::THREADS, P::BYTES, a.stream>>>(a.V, a.lam, a.gV, a.gL, a.gA, a.batch, a.n,
                                                 a.degree, a.status, a.flags);
  return cudaGetLastError();
}

template <int NMAX>
static cudaError_t go_bwd_n(const BwdArgs& a) {
  return a.n == NMAX ? go_bwd<NMAX, true>(a) : go_bwd<NMAX, false>(a);
}

// 33 <= n <= 64 on the tensor cores (bed_backward_tc.cuh); BED_TC=0 selects
// the FFMA2 kernel instead (A/B comparisons)
static bool bwd_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("BED_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

static cudaError_t go_bwd_tc(const BwdArgs& a) {
  auto kern = bed_backward_tc_kernel;
  if (cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), BwdTcParams::BYTES); e != cudaSuccess)
    return e;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t slots = (int64_t)BwdTcParams::CTAS_PER_SM * sms;
  const unsigned grid = (unsigned)(a.batch < slots ? a.batch : slots);
  kern<<<grid, BwdTcParams::THREADS, BwdTcParams::BYTES, a.stream>>>(a.V, a.lam, a.gV, a.gL, a.gA, a.batch,
                                                                    a.n, a.degree, a.status, a.flags);
  return cudaGetLastError();
}

cudaError_t launch_backward(const BwdArgs& a) {
  if (a.n > 32 && bwd_tc_enabled()) return go_bwd_tc(a);
  if (a.n <= 4) return go_bwd_n<4>(a);
  if (a.n <= 8) return go_bwd_n<8>(a);
  if (a.n <= 16) return go_bwd_n<16>(a);
  if (a.n <= 32) return go_bwd_n<32>(a);
  return go_bwd_n<64>(a);
}

}  // namespace bed

// Instantiations of the lane-group forward kernel for the n <= 64 tier.
#include "bed_launch.h"
#include "bed_medium.cuh"

namespace bed {

template <int NMAX, bool EXACT, bool VECS>
static cudaError_t go_medium(const FwdArgs& a) {
  constexpr int T = 4, S = 8;
  using P = MedParams<NMAX, T, S>;
  auto kern = bed_medium_kernel<NMAX, EXACT, VECS, T, S>;
  static bool attr_set = false;  // benign race: idempotent attribute
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)P::BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const unsigned grid = (unsigned)((a.batch + T - 1) / T);
  kern<<<grid, P::THREADS, P::BYTES, a.stream>>>(a.A, a.batch, a.n, a.evals, a.evecs, a.status,
                                                 a.steps, a.flags, a.cfg);
  return cudaGetLastError();
}

template <int NMAX, bool EXACT>
static cudaError_t go_medium_v(const FwdArgs& a) {
  return a.evecs ? go_medium<NMAX, EXACT, true>(a) : go_medium<NMAX, EXACT, false>(a);
}

cudaError_t launch_medium64(const FwdArgs& a) {
  if (a.n == 64) return go_medium_v<64, true>(a);
  if (a.n == 48) return go_medium_v<48, true>(a);
  return go_medium_v<64, false>(a);
}

}  // namespace bed

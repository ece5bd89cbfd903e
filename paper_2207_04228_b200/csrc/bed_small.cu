// Instantiations of the lane-per-matrix forward kernel, n = 1..8.
#include "bed_launch.h"
#include "bed_small.cuh"

namespace bed {

template <int N>
static cudaError_t go_small(const FwdArgs& a) {
  const unsigned grid = (unsigned)((a.batch + kSmallThreads - 1) / kSmallThreads);
  if (a.sc) {  // covariance producer fused in front (and the power behind, if asked)
    const PowSpec pw = a.pw ? *a.pw : PowSpec{};
    if (a.pw)
      bed_small_kernel<N, true, true, true><<<grid, kSmallThreads, 0, a.stream>>>(
          a.A, a.batch, a.evals, a.evecs, a.status, a.steps, a.flags, a.cfg, a.dg, pw, *a.sc);
    else if (a.evecs)
      bed_small_kernel<N, true, false, true><<<grid, kSmallThreads, 0, a.stream>>>(
          a.A, a.batch, a.evals, a.evecs, a.status, a.steps, a.flags, a.cfg, a.dg, pw, *a.sc);
    else
      bed_small_kernel<N, false, false, true><<<grid, kSmallThreads, 0, a.stream>>>(
          a.A, a.batch, a.evals, a.evecs, a.status, a.steps, a.flags, a.cfg, a.dg, pw, *a.sc);
  } else if (a.pw)
    bed_small_kernel<N, true, true><<<grid, kSmallThreads, 0, a.stream>>>(
        a.A, a.batch, a.evals, a.evecs, a.status, a.steps, a.flags, a.cfg, a.dg, *a.pw);
  else if (a.evecs)
    bed_small_kernel<N, true><<<grid, kSmallThreads, 0, a.stream>>>(
        a.A, a.batch, a.evals, a.evecs, a.status, a.steps, a.flags, a.cfg, a.dg);
  else
    bed_small_kernel<N, false><<<grid, kSmallThreads, 0, a.stream>>>(
        a.A, a.batch, a.evals, a.evecs, a.status, a.steps, a.flags, a.cfg, a.dg);
  return cudaGetLastError();
}

cudaError_t launch_small(const FwdArgs& a) {
  switch (a.n) {
    case 1: return go_small<1>(a);
    case 2: return go_small<2>(a);
    case 3: return go_small<3>(a);
    case 4: return go_small<4>(a);
    case 5: return go_small<5>(a);
    case 6: return go_small<6>(a);
    case 7: return go_small<7>(a);
    case 8: return go_small<8>(a);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bed

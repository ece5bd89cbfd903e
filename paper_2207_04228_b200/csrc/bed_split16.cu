// Instantiations of the three-kernel forward for the n <= 16 tier.
#include "bed_split_launch.cuh"

namespace bed {

cudaError_t launch_split16(const FwdArgs& a) {
  if (a.n == 16) return run_split<16, true>(a);
  return run_split<16, false>(a);
}

}  // namespace bed

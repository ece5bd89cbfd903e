// Instantiations of the three-kernel forward for the n <= 64 tier.
#include "bed_split_launch.cuh"

namespace bed {

cudaError_t launch_split64(const FwdArgs& a) {
  if (a.n == 64) return run_split<64, true>(a);
  return run_split<64, false>(a);
}

}  // namespace bed

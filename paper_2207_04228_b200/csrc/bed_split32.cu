// Instantiations of the three-kernel forward for the 25 <= n <= 32 tier.
#include "bed_split_launch.cuh"

namespace bed {

cudaError_t launch_split32(const FwdArgs& a) {
  if (a.n == 32) return run_split<32, true>(a);
  return run_split<32, false>(a);
}

}  // namespace bed

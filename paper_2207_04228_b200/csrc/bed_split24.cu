// Instantiations of the forward for the 17 <= n <= 24 tier (H + fused QF).
#include "bed_split_launch.cuh"

namespace bed {

cudaError_t launch_split24(const FwdArgs& a) {
  if (a.n == 24) return run_split<24, true>(a);
  return run_split<24, false>(a);
}

}  // namespace bed

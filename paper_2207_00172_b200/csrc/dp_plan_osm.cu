// dp_plan_osm.cu -- instantiates the DP kernels for mode DP_PLAN, options in
// shared memory (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_plan_osm(int kmin, int kmax) { return pick_dp_kernel<DP_PLAN, true>(kmin, kmax); }


}  // namespace turbo

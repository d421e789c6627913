// dp_plan.cu -- instantiates the DP kernels for mode DP_PLAN, options in
// registers (shuffle broadcast) (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_plan_reg(int kmin, int kmax) { return pick_dp_kernel<DP_PLAN, false>(kmin, kmax); }
dp_kernel_t dp_kernel_plan_osm(int kmin, int kmax);
dp_kernel_t dp_kernel_plan(int kmin, int kmax, bool osm) { return osm ? dp_kernel_plan_osm(kmin, kmax) : dp_kernel_plan_reg(kmin, kmax); }
}  // namespace turbo

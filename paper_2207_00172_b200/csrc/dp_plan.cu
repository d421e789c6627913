// dp_plan.cu -- instantiates the DP kernels for mode DP_PLAN (split per mode for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_plan(int kmin, int kmax) { return pick_dp_kernel<DP_PLAN>(kmin, kmax); }
}  // namespace turbo

// dp_schedule_global.cu -- fused a1..a6 kernels (turbo_schedule), choice planes in HBM.
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_schedule_global(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_GLOBAL, true, true>(kmin, kmax); }
}  // namespace turbo

// dp_sched_global_reg.cu -- fused a1..a6 kernels (turbo_schedule): choice planes in global,
// options reg (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_sched_global_reg(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_GLOBAL, false, true>(kmin, kmax); }
}  // namespace turbo

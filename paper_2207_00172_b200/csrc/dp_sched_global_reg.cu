// dp_sched_global_reg.cu -- fused a1..a4 kernels of turbo_schedule for windows whose choice
// planes go to HBM: the DP runs in plan mode and the walk (a5) + statistics (a6) follow in
// walk_sched_kernel (backtrack_stats.cu). Options in registers (split per file for
// parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_sched_global_reg(int kmin, int kmax) { return pick_dp_kernel<DP_PLAN, false, true>(kmin, kmax); }
}  // namespace turbo

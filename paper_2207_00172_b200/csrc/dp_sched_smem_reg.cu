// dp_sched_smem_reg.cu -- fused a1..a6 kernels (turbo_schedule): choice planes in smem,
// options reg (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_sched_smem_reg(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_SMEM, false, true>(kmin, kmax); }
}  // namespace turbo

// dp_schedule_smem.cu -- fused a1..a6 kernels (turbo_schedule), choice planes in shared memory.
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_schedule_global(int kmin, int kmax);
dp_kernel_t dp_kernel_schedule(int kmin, int kmax, int mode)
{
    return mode == DP_SOLVE_SMEM ? pick_dp_kernel<DP_SOLVE_SMEM, true, true>(kmin, kmax)
                                 : dp_kernel_schedule_global(kmin, kmax);
}
}  // namespace turbo

// dp_solve_smem.cu -- instantiates the DP kernels for mode DP_SOLVE_SMEM (split per mode for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_solve_smem(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_SMEM>(kmin, kmax); }
}  // namespace turbo

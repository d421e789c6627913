// dp_solve_global.cu -- instantiates the DP kernels for mode DP_SOLVE_GLOBAL (split per mode for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_solve_global(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_GLOBAL>(kmin, kmax); }
}  // namespace turbo

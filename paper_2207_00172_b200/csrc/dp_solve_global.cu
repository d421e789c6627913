// dp_solve_global.cu -- instantiates the DP kernels for mode DP_SOLVE_GLOBAL, options in
// registers (shuffle broadcast) (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_solve_global_reg(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_GLOBAL, false>(kmin, kmax); }
dp_kernel_t dp_kernel_solve_global_osm(int kmin, int kmax);
dp_kernel_t dp_kernel_solve_global(int kmin, int kmax, bool osm) { return osm ? dp_kernel_solve_global_osm(kmin, kmax) : dp_kernel_solve_global_reg(kmin, kmax); }
}  // namespace turbo

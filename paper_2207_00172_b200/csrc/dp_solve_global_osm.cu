// dp_solve_global_osm.cu -- instantiates the DP kernels for mode DP_SOLVE_GLOBAL, options in
// shared memory (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_solve_global_osm(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_GLOBAL, true>(kmin, kmax); }


}  // namespace turbo

// dp_solve_smem_osm.cu -- instantiates the DP kernels for mode DP_SOLVE_SMEM, options in
// shared memory (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_solve_smem_osm(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_SMEM, true>(kmin, kmax); }


}  // namespace turbo

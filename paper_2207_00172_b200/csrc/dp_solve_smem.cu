// dp_solve_smem.cu -- instantiates the DP kernels for mode DP_SOLVE_SMEM, options in
// registers (shuffle broadcast) (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_solve_smem_reg(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_SMEM, false>(kmin, kmax); }
dp_kernel_t dp_kernel_solve_smem_osm(int kmin, int kmax);
dp_kernel_t dp_kernel_solve_smem(int kmin, int kmax, bool osm) { return osm ? dp_kernel_solve_smem_osm(kmin, kmax) : dp_kernel_solve_smem_reg(kmin, kmax); }
}  // namespace turbo

// dp_sched_global_osm.cu -- fused a1..a6 kernels (turbo_schedule): choice planes in global,
// options osm (split per file for parallel builds).
#include "dp_kernel.cuh"

namespace turbo {
dp_kernel_t dp_kernel_sched_global_osm(int kmin, int kmax) { return pick_dp_kernel<DP_SOLVE_GLOBAL, true, true>(kmin, kmax); }
}  // namespace turbo

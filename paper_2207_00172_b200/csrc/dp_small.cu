// dp_small.cu -- the fixed-K fused-solve kernels (choice planes in shared memory, options staged,
// walk in the kernel) for launches of at most 4 warps per window (rows of <= 4 tiles: c1, c2):
// __launch_bounds__(128, 7) gives them 72 registers, so the frame loop keeps its invariants in
// registers instead of re-deriving them every frame under the 64-register budget of the 512-thread
// instantiations. nullptr: no such kernel for this K range (the general kernels serve it).
#include "dp_kernel.cuh"

namespace turbo {

template <bool FUSE>
static dp_kernel_t pick_small(int kmin, int kmax)
{
    if (kmin != kmax) return nullptr;
    switch (kmin) {
        case 4: return dp_cta_kernel<4, DP_SOLVE_SMEM, true, FUSE, false, true>;
        case 5: return dp_cta_kernel<5, DP_SOLVE_SMEM, true, FUSE, false, true>;
        case 6: return dp_cta_kernel<6, DP_SOLVE_SMEM, true, FUSE, false, true>;
        case 8: return dp_cta_kernel<8, DP_SOLVE_SMEM, true, FUSE, false, true>;
        default: return nullptr;
    }
}

dp_kernel_t dp_kernel_small(int kmin, int kmax, bool fuse)
{
    return fuse ? pick_small<true>(kmin, kmax) : pick_small<false>(kmin, kmax);
}

}  // namespace turbo

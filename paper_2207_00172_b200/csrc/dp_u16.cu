// dp_u16.cu -- NEXT-5: the fixed-K fused-solve kernels (choice planes in shared
// memory, options staged, walk in the kernel) that plan qualifying windows on u16 rows
// (dp_kernel.cuh dp_tile_u16); opt-in with turbo_debug_set_variant bit 128. nullptr: no u16 kernel
// for this K range (the int32 kernels serve it).
#include "dp_kernel.cuh"

namespace turbo {

template <bool FUSE>
static dp_kernel_t pick_u16(int kmin, int kmax)
{
    if (kmin != kmax) return nullptr;
    switch (kmin) {
        case 4: return dp_cta_kernel<4, DP_SOLVE_SMEM, true, FUSE, true>;
        case 5: return dp_cta_kernel<5, DP_SOLVE_SMEM, true, FUSE, true>;
        case 6: return dp_cta_kernel<6, DP_SOLVE_SMEM, true, FUSE, true>;
        case 8: return dp_cta_kernel<8, DP_SOLVE_SMEM, true, FUSE, true>;
        default: return nullptr;
    }
}

dp_kernel_t dp_kernel_u16(int kmin, int kmax, bool fuse)
{
    return fuse ? pick_u16<true>(kmin, kmax) : pick_u16<false>(kmin, kmax);
}

}  // namespace turbo

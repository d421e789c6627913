// dp_gen.cu -- the mixed-K plan-mode DP launches of the short-row classes: one runtime-K body
// (dp_window_gen in dp_kernel.cuh), one CTA of G warps per window, compiled with a 64-register
// cap. Those windows are latency-bound chains (a few tiles per frame), so what they need is
// many resident warps and a small instruction footprint: the K-specific mixed kernel
// (dp_cta_kernel<0>) carries fifteen unrolled bodies and 128 registers per thread, which held
// c5's row class 1 to 16 warps per SM and thrashed the instruction cache (ncu: 37 / 10.5
// "no instruction" stalls per issued instruction in classes 0 / 1).
#include "dp_kernel.cuh"

namespace turbo {

// SMALL: launches of <= 4 warps per window (row classes 0-1): 72 registers (7 x 128 threads / SM)
template <bool OSM, bool FUSE, bool SMALL = false>
__global__ void __launch_bounds__(SMALL ? 128 : 512, SMALL ? 7 : 2) dp_gen_kernel(DpParams P)
{
    extern __shared__ int4 smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    int64_t *red = reinterpret_cast<int64_t *>(smem_raw);
    int32_t *base = reinterpret_cast<int32_t *>(smem_raw) + 16;
    const int32_t stride = P.pad_words + P.row_words;
    int32_t *rowA = base + P.pad_words;
    int32_t *rowB = rowA + stride;
    int2 *opt_s = reinterpret_cast<int2 *>(base + (nwarps > 1 ? 2 : 1) * stride);
    for (int32_t x = threadIdx.x; x < P.pad_words; x += blockDim.x) {
        rowA[x - P.pad_words] = NEG_R;
        if (nwarps > 1) rowB[x - P.pad_words] = NEG_R;
    }
    __syncthreads();
    const int64_t n = P.ordered ? (int64_t)P.cls_count : (int64_t)P.num_windows;
    for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
        int64_t w = r;
        if (P.ordered) {
            w = P.windows[P.cls_first + r].order;
        } else {
            const int rc = row_class((int64_t)P.windows[w].budget_bound + 1);
            if (rc >= TURBO_NUM_CLASSES || (P.cls >= 0 && rc != P.cls)) continue;
        }
        const int K = P.windows[w].num_exits;
        if (K <= 4)
            dp_window_gen<2, OSM, FUSE>(P, w, K, rowA, rowB, opt_s, red, warp, nwarps, lane);
        else
            dp_window_gen<4, OSM, FUSE>(P, w, K, rowA, rowB, opt_s, red, warp, nwarps, lane);
        __syncthreads();                              // smem reused by the next window
    }
}

dp_kernel_t dp_kernel_generic(bool osm, bool fuse, bool small)
{
    if (small) {             // same-box A/B, c5: 13.28 -> 13.20 ms
        if (fuse) return osm ? dp_gen_kernel<true, true, true> : dp_gen_kernel<false, true, true>;
        return osm ? dp_gen_kernel<true, false, true> : dp_gen_kernel<false, false, true>;
    }
    if (fuse) return osm ? dp_gen_kernel<true, true> : dp_gen_kernel<false, true>;
    return osm ? dp_gen_kernel<true, false> : dp_gen_kernel<false, false>;
}

}  // namespace turbo

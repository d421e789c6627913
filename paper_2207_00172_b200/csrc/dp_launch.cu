// dp_launch.cu -- launch configuration of the DP kernels (dp_kernel.cuh).
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "dp_kernel.cuh"

namespace turbo {

// Windows resident per SM, s. Equal windows finish in waves; when the SM is throughput-bound a
// wave of s windows costs ~s, so ceil(W / (num_sms * s)) * s measures the partly filled last
// wave. More resident warps also hide latency, so take the LARGEST s whose cost is within 5%
// of the minimum.
static int pick_concurrency(int64_t W, int num_sms, int s_max)
{
    int64_t best_cost = INT64_MAX;
    for (int s = 1; s <= s_max; ++s) {
        const int64_t slots = (int64_t)num_sms * s;
        const int64_t cost = ((W + slots - 1) / slots) * s;
        if (cost < best_cost) best_cost = cost;
    }
    for (int s = s_max; s >= 1; --s) {
        const int64_t slots = (int64_t)num_sms * s;
        const int64_t cost = ((W + slots - 1) / slots) * s;
        if (cost * 100 <= best_cost * 105) return s;
    }
    return 1;
}

// Warps per window: one warp (in-place row) when the row is a single tile, else up to 8
// warps sharing the tiles (double-buffered row).
int dp_warps_per_window(const turbo_shape_t *s)
{
    const int rpt = s->max_exits <= 4 ? 16 : 8;
    const int64_t tiles = (num_rows(s->max_budget_small) + rpt - 1) / rpt;
    static int forced = -1;
    if (forced < 0) {
        const char *e = getenv("TURBO_DP_WARPS");          // tuning override (1, 2, 4, 8)
        forced = e ? atoi(e) : 0;
    }
    if (forced > 0 && tiles > 1) return forced > 16 ? 16 : forced;
    if (tiles <= 1) return 1;
    if (tiles >= 32) return 16;      // long rows: more warps per SM to hide LDS/barrier latency
    return tiles >= 8 ? 8 : (int)tiles;
}

static cudaError_t prepare(dp_kernel_t kern, size_t smem)
{
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> limit;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(dev, (const void *)kern);
    auto it = limit.find(key);
    if (it == limit.end()) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                             (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        it = limit.emplace(key, 0).first;
    }
    if (smem > it->second) {     // the attribute call is not free: only when the need grows
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        it->second = smem;
    }
    return cudaSuccess;
}

size_t dp_smem_bytes(const DpParams &P, int nwarps)
{
    return 64 + (size_t)4 * ((size_t)(nwarps > 1 ? 2 : 1) * (P.pad_words + P.row_words) + P.chs_words +
                             P.cst_words);
}

// The kernel a class launch uses, and its dynamic-smem ceiling (the per-CTA opt-in maximum minus
// the kernel's static smem). Host-only queries: run_dp calls this for every class BEFORE any launch.
static cudaError_t resolve_dp(const turbo_shape_t *shape, int mode, const DpParams &P, int smem_per_cta_max,
                              dp_kernel_t *kern_out, size_t *dyn_max_out)
{
    const bool osm = P.osm != 0;
    // (HBM choice planes are always walked by a separate kernel: DP_SOLVE_GLOBAL never gets here)
    if (mode == DP_SOLVE_GLOBAL) return cudaErrorInvalidValue;
    if (P.generic && mode != DP_PLAN) return cudaErrorInvalidValue;
    // NEXT-5 u16 rows (opt-in, P.u16): the fixed-K fused-solve kernels with staged options
    dp_kernel_t kern = (P.u16 && osm && mode == DP_SOLVE_SMEM && !P.generic)
                           ? dp_kernel_u16(shape->min_exits, shape->max_exits, P.fuse != 0)
                           : nullptr;
    // launches of <= 4 warps per window: the 72-register instantiations (dp_small.cu)
    if (kern == nullptr && osm && mode == DP_SOLVE_SMEM && !P.generic && dp_warps_per_window(shape) <= 4 &&
        P.small)
        kern = dp_kernel_small(shape->min_exits, shape->max_exits, P.fuse != 0);
    if (kern == nullptr)
        kern = P.generic               ? dp_kernel_generic(osm, P.fuse != 0, dp_warps_per_window(shape) <= 4 && P.small)
               : P.fuse                ? dp_kernel_schedule(shape->min_exits, shape->max_exits, mode, osm)
               : mode == DP_PLAN         ? dp_kernel_plan(shape->min_exits, shape->max_exits, osm)
                                         : dp_kernel_solve_smem(shape->min_exits, shape->max_exits, osm);
    static std::mutex amu;
    static std::map<const void *, size_t> static_smem;
    size_t st_bytes = 0;
    {
        std::lock_guard<std::mutex> lk(amu);
        auto it = static_smem.find((const void *)kern);
        if (it == static_smem.end()) {
            cudaFuncAttributes fa;
            cudaError_t e = cudaFuncGetAttributes(&fa, kern);
            if (e != cudaSuccess) return e;
            it = static_smem.emplace((const void *)kern, fa.sharedSizeBytes).first;
        }
        st_bytes = it->second;
    }
    if ((size_t)smem_per_cta_max <= st_bytes) return cudaErrorInvalidConfiguration;
    *kern_out = kern;
    *dyn_max_out = (size_t)smem_per_cta_max - st_bytes;
    return cudaSuccess;
}

cudaError_t check_dp(const turbo_shape_t *shape, int mode, const DpParams &P, int smem_per_cta_max)
{
    dp_kernel_t kern = nullptr;
    size_t dyn_max = 0;
    cudaError_t e = resolve_dp(shape, mode, P, smem_per_cta_max, &kern, &dyn_max);
    if (e != cudaSuccess) return e;
    return dp_smem_bytes(P, dp_warps_per_window(shape)) > dyn_max ? cudaErrorInvalidConfiguration : cudaSuccess;
}

cudaError_t launch_dp(const turbo_shape_t *shape, int mode, const DpParams &P0, int num_sms, int smem_per_sm,
                      int smem_per_cta_max, cudaStream_t stream, DpLaunch *info)
{
    DpParams P = P0;
    const int64_t W = shape->num_windows;
    if (W <= 0) return cudaSuccess;
    const int G = dp_warps_per_window(shape);
    P.warps_per_cta = G;
    const size_t need = dp_smem_bytes(P, G);
    dp_kernel_t kern = nullptr;
    size_t dyn_max = 0;
    cudaError_t e = resolve_dp(shape, mode, P, smem_per_cta_max, &kern, &dyn_max);
    if (e != cudaSuccess) return e;
    if (need > dyn_max) return cudaErrorInvalidConfiguration;
    e = prepare(kern, dyn_max);
    if (e != cudaSuccess) return e;
    // s_max from the occupancy calculator (it knows the per-CTA reservation and the carveout);
    // results are cached per (device, kernel, G, need, W) -- the queries are host-side only
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int, size_t, int64_t>, size_t> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const int64_t Wc = P.cls_count > 0 ? P.cls_count : W;   // windows this launch plans
    const auto ckey = std::make_tuple(dev, (const void *)kern, G, need, Wc);
    size_t smem = need;
    bool cached = false;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(ckey);
        if (it != cache.end()) {
            smem = it->second;
            cached = true;
        }
    }
    int s_max = 0;
    if (!cached) {
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s_max, kern, 32 * G, need);
        if (e != cudaSuccess) return e;
        if (s_max < 1) return cudaErrorInvalidConfiguration;
    }
    const int s = cached ? 0 : pick_concurrency(Wc, num_sms, s_max);
    // pad the dynamic smem so that exactly s CTAs fit per SM (occupancy as a knob)
    if (!cached && s < s_max) {
        size_t hi = dyn_max, lo = need;                       // largest smem with occupancy >= s
        while (hi - lo > 16) {
            const size_t mid = ((lo + hi) / 2) & ~(size_t)15;
            int occ = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * G, mid);
            if (e != cudaSuccess) return e;
            if (occ >= s) lo = mid; else hi = mid;
        }
        smem = lo;
    }
    if (!cached) {
        std::lock_guard<std::mutex> lk(mu);
        cache[ckey] = smem;
    }
    const int64_t blocks = P.ordered ? (int64_t)P.cls_count : W;
    if (blocks <= 0) return cudaSuccess;
    note_launch();
    kern<<<(unsigned)blocks, 32 * G, smem, stream>>>(P);
    if (info) {
        info->mode = mode;
        info->warps_per_cta = G;
        info->blocks = (int)blocks;
        info->smem_bytes = smem;
    }
    return cudaGetLastError();
}

}  // namespace turbo

namespace turbo {
dp_kernel_t dp_kernel_generic(bool osm, bool fuse, bool small);
dp_kernel_t dp_kernel_sched_smem_osm(int kmin, int kmax);
dp_kernel_t dp_kernel_sched_smem_reg(int kmin, int kmax);
dp_kernel_t dp_kernel_sched_global_osm(int kmin, int kmax);
dp_kernel_t dp_kernel_sched_global_reg(int kmin, int kmax);
dp_kernel_t dp_kernel_schedule(int kmin, int kmax, int mode, bool osm)
{
    if (mode == DP_SOLVE_SMEM) return osm ? dp_kernel_sched_smem_osm(kmin, kmax) : dp_kernel_sched_smem_reg(kmin, kmax);
    // DP_PLAN: fused a1..a4, the walk and statistics follow in walk_sched_kernel
    return osm ? dp_kernel_sched_global_osm(kmin, kmax) : dp_kernel_sched_global_reg(kmin, kmax);
}
}  // namespace turbo

// lookup.cu -- K1: window budget (a1) + class -> profile gather (a2). HBM-bound.
//
// a1 (§3 "quantifying the number of frames reaching the object detector";
//     reading R3): budget_w = max(0, capacity_w - m_w * u0).
// a2 (PAPER.md:511 §5.1 accuracy profile P_k^theta per bucket; :502-509 latency I_k;
//     :519-525 §5.2 the per-frame terms of the objective and constraint):
//     opt_gain[x][k] = gain[class_x][k], opt_cost[x][k] = cost[class_x][k].
//
// One warp per (window, chunk of LK_CHUNK option vectors): long windows (c4: 4,500 vectors) are
// spread over many warps instead of one latency-bound warp, short ones take one chunk.
// turbo_mckp_workspace pads every window's option block to a multiple of 4 int32 and aligns it
// to 16 B, so each lane writes whole int4 vectors: per option 8 B of coalesced 16-B stores, per
// frame 1 B of class id (broadcast to K lanes).
#include <algorithm>

#include "turbo_internal.cuh"

namespace turbo {

constexpr int LK_CHUNK = 256;                        // option vectors (of 4) per warp task

__global__ void __launch_bounds__(256) lookup_kernel(const turbo_profile_t *__restrict__ profiles,
                                                     turbo_window_t *__restrict__ windows, int32_t num_windows,
                                                     const uint8_t *__restrict__ class_id,
                                                     const int32_t *__restrict__ capacity, int32_t base_cost,
                                                     int32_t *__restrict__ opt_gain, int32_t *__restrict__ opt_cost,
                                                     int64_t *__restrict__ status, int32_t chunks_per_window)
{
    const int lane = threadIdx.x & 31;
    const int warps_per_cta = blockDim.x >> 5;
    const int64_t ntask = (int64_t)num_windows * chunks_per_window;
    for (int64_t task = (int64_t)blockIdx.x * warps_per_cta + (threadIdx.x >> 5); task < ntask;
         task += (int64_t)gridDim.x * warps_per_cta) {
        const int64_t w = task / chunks_per_window;
        const int32_t chunk = (int32_t)(task - w * chunks_per_window);
        const int64_t ff = windows[w].first_frame;
        const int64_t fo = windows[w].first_option;
        const int32_t N = windows[w].num_frames;
        const int32_t p = windows[w].profile;
        if (capacity != nullptr && lane == 0 && chunk == 0) {
            int64_t b = (int64_t)capacity[w] - (int64_t)N * (int64_t)base_cost;   // a1
            windows[w].budget = (int32_t)(b < 0 ? 0 : b);
        }
        const int32_t C = profiles[p].num_classes;
        const int32_t K = profiles[p].num_exits;
        const int32_t *__restrict__ pg = profiles[p].gain;
        const int32_t *__restrict__ pc = profiles[p].cost;
        // exact o / K for o < 2^20 via a 32-bit reciprocal (K <= 16)
        const uint32_t magic = (uint32_t)((0x100000000ull + (uint64_t)K - 1) / (uint64_t)K);
        const int32_t n_opt = N * K;
        const int32_t n_vec = (n_opt + 3) >> 2;
        int4 *__restrict__ dg = reinterpret_cast<int4 *>(opt_gain + fo);
        int4 *__restrict__ dc = reinterpret_cast<int4 *>(opt_cost + fo);
        const int32_t v_end = min(n_vec, (chunk + 1) * LK_CHUNK);
        for (int32_t v = chunk * LK_CHUNK + lane; v < v_end; v += 32) {
            int32_t gv[4], cv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t o = (uint32_t)(v * 4 + e);
                const uint32_t i = __umulhi(o, magic);
                const uint32_t k = o - i * (uint32_t)K;
                gv[e] = 0;
                cv[e] = 0;
                if ((int32_t)o < n_opt) {
                    const int32_t cls = class_id[ff + i];
                    if (cls < C) {
                        gv[e] = __ldg(pg + cls * K + k);
                        cv[e] = __ldg(pc + cls * K + k);
                    } else if (k == 0) {
                        atomic_min_i64(&status[0], ff + i);
                    }
                }
            }
            dg[v] = make_int4(gv[0], gv[1], gv[2], gv[3]);
            dc[v] = make_int4(cv[0], cv[1], cv[2], cv[3]);
        }
    }
}

cudaError_t launch_lookup(const turbo_profile_t *profiles, turbo_window_t *windows, int32_t num_windows,
                          const uint8_t *class_id, const int32_t *capacity, int32_t base_cost, int32_t *opt_gain,
                          int32_t *opt_cost, int64_t *status, int32_t max_options, int num_sms, cudaStream_t stream)
{
    if (num_windows <= 0) return cudaSuccess;
    const int threads = 256;
    const int warps = threads / 32;
    const int32_t cpw = std::max(1, (int32_t)(((int64_t)max_options + 4 * LK_CHUNK - 1) / (4 * LK_CHUNK)));
    int64_t blocks = ((int64_t)num_windows * cpw + warps - 1) / warps;
    const int64_t cap = (int64_t)num_sms * 16;
    if (blocks > cap) blocks = cap;
    note_launch();
    lookup_kernel<<<(unsigned)blocks, threads, 0, stream>>>(profiles, windows, num_windows, class_id, capacity,
                                                            base_cost, opt_gain, opt_cost, status, cpw);
    return cudaGetLastError();
}

}  // namespace turbo

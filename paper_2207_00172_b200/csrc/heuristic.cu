// heuristic.cu -- NEXT-1: the paper's own scheduler, prune-and-search (§5.2),
// batched over windows as a comparison arm for the exact DP (the paper's "upper", :858 §6.4).
//
//   1) every frame starts at the maximum level kappa = K-1;
//   2) while the plan's cost exceeds the budget, the frame with the minimal marginal accuracy
//      gain g_{i,k} - g_{i,k-1} is downgraded to k-1 (ties: larger latency reduction
//      c_{i,k} - c_{i,k-1} first, then smaller frame id -- SPEC.md:263-271);
//   3) stop when the cost fits, or every frame is at level 0 (then feasible = 0).
// With per-frame additive costs (reading R1) the cost is sum_i c_{i,k_i}.
//
// B200 mapping: one warp per window. The levels live in shared memory (one byte per frame);
// each lane owns frames lane, lane+32, ... and keeps the best (key, id) among them; a step is a
// 5-round shuffle argmin over the warp, after which only the winning lane rescans its frames.
#include <climits>

#include "turbo_internal.cuh"

namespace turbo {

struct HeurParams {
    const turbo_window_t *windows;
    int32_t num_windows;
    int32_t frames_cap;            // bytes of level storage per warp
    const int32_t *opt_gain;
    const int32_t *opt_cost;
    int32_t *gain_out;
    int32_t *cost_out;
    uint8_t *feasible;
    uint8_t *exit_out;
    int32_t *steps;
};

__device__ __forceinline__ void heur_key(const int32_t *og, const int32_t *oc, int K, int32_t i, int k,
                                         long long &key)
{
    if (k == 0) {
        key = LLONG_MAX;                             // cannot be downgraded
        return;
    }
    const int32_t m = __ldg(og + (int64_t)i * K + k) - __ldg(og + (int64_t)i * K + k - 1);
    const int32_t dc = __ldg(oc + (int64_t)i * K + k) - __ldg(oc + (int64_t)i * K + k - 1);
    // order: smaller marginal gain, then larger latency reduction (the frame id breaks the rest)
    key = (long long)m * 4294967296ll + (long long)(uint32_t)(0x7fffffff - dc);
}

__global__ void __launch_bounds__(256) heuristic_kernel(HeurParams P)
{
    extern __shared__ uint8_t lv_all[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int wpc = blockDim.x >> 5;
    uint8_t *lv = lv_all + (size_t)warp * P.frames_cap;
    for (int64_t w = (int64_t)blockIdx.x * wpc + warp; w < P.num_windows; w += (int64_t)gridDim.x * wpc) {
        const turbo_window_t &win = P.windows[w];
        const int32_t N = win.num_frames, K = win.num_exits, B = win.budget;
        const int32_t *og = P.opt_gain + win.first_option;
        const int32_t *oc = P.opt_cost + win.first_option;
        // 1) all frames at K-1
        long long cost = 0;
        for (int32_t i = lane; i < N; i += 32) {
            lv[i] = (uint8_t)(K - 1);
            cost += __ldg(oc + (int64_t)i * K + K - 1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cost += __shfl_xor_sync(0xffffffffu, cost, o);
        __syncwarp();
        auto rescan = [&](long long &bk, int32_t &bi) {
            bk = LLONG_MAX;
            bi = INT32_MAX;
            for (int32_t i = lane; i < N; i += 32) {
                long long k;
                heur_key(og, oc, K, i, lv[i], k);
                if (k < bk) {                             // ids ascend within a lane: strict keeps the smaller
                    bk = k;
                    bi = i;
                }
            }
        };
        long long my_key;
        int32_t my_id;
        rescan(my_key, my_id);
        int32_t steps = 0;
        // 2) downgrade the minimal-marginal frame until the plan fits
        while (cost > B) {
            long long k = my_key;
            int32_t id = my_id;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const long long k2 = __shfl_xor_sync(0xffffffffu, k, o);
                const int32_t id2 = __shfl_xor_sync(0xffffffffu, id, o);
                if (k2 < k || (k2 == k && id2 < id)) {
                    k = k2;
                    id = id2;
                }
            }
            if (k == LLONG_MAX) break;                    // 3) every frame at level 0
            const long long dc = 0x7fffffffll - (long long)(uint32_t)(k & 0xffffffffll);   // may be < 0
            cost -= dc;
            steps += 1;
            if ((id & 31) == lane) {
                lv[id] = (uint8_t)(lv[id] - 1);
                rescan(my_key, my_id);
            }
            __syncwarp();
        }
        long long gain = 0;
        for (int32_t i = lane; i < N; i += 32) {
            const int k = lv[i];
            gain += __ldg(og + (int64_t)i * K + k);
            P.exit_out[win.first_frame + i] = (uint8_t)k;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) gain += __shfl_xor_sync(0xffffffffu, gain, o);
        if (lane == 0) {
            P.gain_out[w] = (int32_t)gain;
            P.cost_out[w] = (int32_t)cost;
            P.feasible[w] = cost <= B ? 1 : 0;
            if (P.steps) P.steps[w] = steps;
        }
        __syncwarp();
    }
}

cudaError_t launch_heuristic(const turbo_shape_t *shape, const turbo_window_t *windows, const int32_t *opt_gain,
                             const int32_t *opt_cost, int32_t *gain_out, int32_t *cost_out, uint8_t *feasible,
                             uint8_t *exit_out, int32_t *steps, int num_sms, int smem_per_cta_max,
                             cudaStream_t stream)
{
    if (shape->num_windows <= 0) return cudaSuccess;
    HeurParams P;
    P.windows = windows;
    P.num_windows = shape->num_windows;
    P.frames_cap = (shape->max_frames + 15) & ~15;
    P.opt_gain = opt_gain;
    P.opt_cost = opt_cost;
    P.gain_out = gain_out;
    P.cost_out = cost_out;
    P.feasible = feasible;
    P.exit_out = exit_out;
    P.steps = steps;
    int wpc = 8;
    while (wpc > 1 && (size_t)wpc * P.frames_cap > (size_t)smem_per_cta_max) wpc >>= 1;
    const size_t smem = (size_t)wpc * P.frames_cap;
    if (smem > (size_t)smem_per_cta_max) return cudaErrorInvalidConfiguration;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(heuristic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    int64_t blocks = ((int64_t)shape->num_windows + wpc - 1) / wpc;
    if (blocks > (int64_t)num_sms * 64) blocks = (int64_t)num_sms * 64;
    note_launch();
    heuristic_kernel<<<(unsigned)blocks, 32 * wpc, smem, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace turbo

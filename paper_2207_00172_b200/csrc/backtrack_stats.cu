// backtrack_stats.cu -- K6 (plan reconstruction, a5) and K7 (plan statistics, a6).
#include "dp_kernel.cuh"

namespace turbo {

// ---------------------------------------------------------------------------------------------
// K6 (a5). Forward walk from (frame 0, b = C*): k_i = choice_i[b]; b -= c_{i,k_i}
// (the realisation of the lexicographic tie-break, reading R7; "we
// execute each frame according to the plan"). The chain of N dependent loads is latency-bound,
// so one warp serves one window and SPECULATES (backtrack_warp_rt): while frame i's word is in
// flight the lanes already fetch frame i+1's (and, for K <= 5, frame i+2's) words for every
// possible shift (costs of frame i do not depend on b), so each round trip resolves 2-3 frames.
__global__ void __launch_bounds__(256) backtrack_kernel(const turbo_window_t *__restrict__ windows,
                                                        int32_t num_windows,
                                                        const int32_t *__restrict__ opt_cost,
                                                        const uint8_t *__restrict__ workspace,
                                                        const int32_t *__restrict__ best_cost,
                                                        const uint8_t *__restrict__ feasible,
                                                        uint8_t *__restrict__ exit_out, WinSel sel)
{
    const int lane = threadIdx.x & 31;
    const int wpc = blockDim.x >> 5;
    for (int64_t r = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); r < sel.n_iter(num_windows);
         r += (int64_t)gridDim.x * wpc) {
        const int64_t w = sel.window(windows, r);
        if (w < 0) continue;
        const int64_t ff = windows[w].first_frame;
        const int64_t fo = windows[w].first_option;
        const int32_t N = windows[w].num_frames;
        const int32_t K = windows[w].num_exits;
        const int32_t Bb = windows[w].budget_bound;
        const uint32_t *__restrict__ gch =
            reinterpret_cast<const uint32_t *>(workspace + windows[w].choice_offset);
        if (!feasible[w]) {
            for (int32_t i = lane; i < N; i += 32) exit_out[ff + i] = 0;
            continue;
        }
        const int RPT = K <= 4 ? 16 : 8;
        const int32_t gtiles = (((Bb + 32) >> 5) + RPT - 1) / RPT;
        const int32_t *__restrict__ oc = opt_cost + fo;
        auto cost = [&](int32_t i, int32_t k) -> int32_t { return __ldg(oc + (int64_t)i * K + k); };
        backtrack_warp_rt(K, N, best_cost[w], gch, gtiles, cost, exit_out + ff, lane);
    }
}

cudaError_t launch_backtrack(const turbo_window_t *windows, int32_t num_windows, const int32_t *opt_cost,
                             const uint8_t *workspace, const int32_t *best_cost, const uint8_t *feasible,
                             uint8_t *exit_out, int num_sms, cudaStream_t stream, WinSel sel)
{
    if (sel.n_iter(num_windows) <= 0) return cudaSuccess;
    const int threads = 128;
    const int wpc = threads / 32;
    int64_t blocks = (sel.n_iter(num_windows) + wpc - 1) / wpc;
    const int64_t cap = (int64_t)num_sms * 16;
    if (blocks > cap) blocks = cap;
    note_launch();
    backtrack_kernel<<<(unsigned)blocks, threads, 0, stream>>>(windows, num_windows, opt_cost, workspace,
                                                               best_cost, feasible, exit_out, sel);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// K6 + K7 of turbo_schedule for the windows whose DP ran in plan mode (choice planes in HBM):
// one warp walks one window (costs straight from its class ids and the profile, as the fused DP
// staged them), then the warp adds the window's plan to the CTA-private statistics, flushed with
// one atomic per non-zero counter at the end. Running the walks here (thousands in flight) frees
// the DP kernel's CTA slots, which an in-kernel walk of HBM planes would hold for its whole
// latency-bound chain.
__global__ void __launch_bounds__(128) walk_sched_kernel(const turbo_window_t *__restrict__ windows,
                                                         int32_t num_windows,
                                                         const turbo_profile_t *__restrict__ profiles,
                                                         const uint8_t *__restrict__ class_id,
                                                         const uint8_t *__restrict__ workspace,
                                                         const int32_t *__restrict__ best_gain,
                                                         const int32_t *__restrict__ best_cost,
                                                         const uint8_t *__restrict__ feasible,
                                                         uint8_t *__restrict__ exit_out,
                                                         unsigned long long *__restrict__ stats, WinSel sel)
{
    __shared__ unsigned int hist[176];
    __shared__ unsigned long long tot[5];
    for (int x = threadIdx.x; x < 176; x += blockDim.x) hist[x] = 0;
    if (threadIdx.x < 5) tot[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wpc = blockDim.x >> 5;
    long long sg = 0, sc = 0, nw = 0, nf = 0, ni = 0;
    for (int64_t r = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); r < sel.n_iter(num_windows);
         r += (int64_t)gridDim.x * wpc) {
        const int64_t w = sel.window(windows, r);
        if (w < 0) continue;
        const turbo_window_t win = windows[w];
        const int64_t ff = win.first_frame;
        const int32_t N = win.num_frames;
        const bool feas = feasible[w] != 0;
        if (!feas) {
            for (int32_t i = lane; i < N; i += 32) exit_out[ff + i] = 0;
        } else {
            const turbo_profile_t pr = profiles[win.profile];
            const int32_t K = pr.num_exits;
            const int RPT = K <= 4 ? 16 : 8;
            const int32_t gtiles = (((win.budget_bound + 32) >> 5) + RPT - 1) / RPT;
            const uint32_t *__restrict__ gch = reinterpret_cast<const uint32_t *>(workspace + win.choice_offset);
            const int32_t b = best_cost[w];
            // one runtime-K walk for every window (a per-K switch of unrolled walks thrashed the
            // instruction cache when neighbouring warps walk windows of different K)
            const uint8_t *__restrict__ cls_ids = class_id + ff;
            const int32_t *__restrict__ prof_c = pr.cost;
            const int32_t C = pr.num_classes;
            auto cost = [&](int32_t i, int32_t k) -> int32_t {
                const int32_t c = cls_ids[i];
                return c < C ? __ldg(prof_c + c * K + k) : 0;
            };
            backtrack_warp_rt(K, N, b, gch, gtiles, cost, exit_out + ff, lane);
        }
        __syncwarp();                                   // lane 0's exit stores -> the warp
        for (int32_t i = lane; i < N; i += 32) {
            const uint32_t k = exit_out[ff + i] & 15u;
            const uint32_t c = class_id[ff + i];
            atomicAdd(&hist[k], 1u);
            if (c < 10) atomicAdd(&hist[16 + c * 16 + k], 1u);
        }
        if (lane == 0) {
            sg += best_gain[w];
            sc += best_cost[w];
            nw += 1;
            nf += N;
            ni += feas ? 0 : 1;
        }
    }
    if (lane == 0) {
        atomicAdd(&tot[0], (unsigned long long)sg);
        atomicAdd(&tot[1], (unsigned long long)sc);
        atomicAdd(&tot[2], (unsigned long long)nw);
        atomicAdd(&tot[3], (unsigned long long)nf);
        atomicAdd(&tot[4], (unsigned long long)ni);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < 176; x += blockDim.x)
        if (hist[x]) atomicAdd(&stats[x], (unsigned long long)hist[x]);
    if (threadIdx.x < 5 && tot[threadIdx.x]) atomicAdd(&stats[176 + threadIdx.x], tot[threadIdx.x]);
}

cudaError_t launch_walk_sched(const turbo_window_t *windows, int32_t num_windows, const turbo_profile_t *profiles,
                              const uint8_t *class_id, const uint8_t *workspace, const int32_t *best_gain,
                              const int32_t *best_cost, const uint8_t *feasible, uint8_t *exit_out, int64_t *stats,
                              int num_sms, cudaStream_t stream, WinSel sel)
{
    if (sel.n_iter(num_windows) <= 0) return cudaSuccess;
    const int threads = 128;
    const int wpc = threads / 32;
    int64_t blocks = (sel.n_iter(num_windows) + wpc - 1) / wpc;
    const int64_t cap = (int64_t)num_sms * 16;
    if (blocks > cap) blocks = cap;
    note_launch();
    walk_sched_kernel<<<(unsigned)blocks, threads, 0, stream>>>(windows, num_windows, profiles, class_id, workspace,
                                                                best_gain, best_cost, feasible, exit_out,
                                                                reinterpret_cast<unsigned long long *>(stats), sel);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// K7 (a6). Per-GPU statistics of the plans, int64[181] (layout in turbo.h): CTA-private
// shared-memory histograms, one global atomic per counter per CTA at the end.
__global__ void __launch_bounds__(256) stats_kernel(const turbo_window_t *__restrict__ windows,
                                                    int32_t num_windows, const uint8_t *__restrict__ class_id,
                                                    const uint8_t *__restrict__ exit_out,
                                                    const int32_t *__restrict__ best_gain,
                                                    const int32_t *__restrict__ best_cost,
                                                    const uint8_t *__restrict__ feasible,
                                                    unsigned long long *__restrict__ stats)
{
    __shared__ unsigned int hist[176];
    __shared__ unsigned long long tot[5];
    for (int x = threadIdx.x; x < 176; x += blockDim.x) hist[x] = 0;
    if (threadIdx.x < 5) tot[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int wpc = blockDim.x >> 5;
    long long sg = 0, sc = 0, nw = 0, nf = 0, ni = 0;
    for (int64_t w = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); w < num_windows;
         w += (int64_t)gridDim.x * wpc) {
        const int64_t ff = windows[w].first_frame;
        const int32_t N = windows[w].num_frames;
        for (int32_t i = lane; i < N; i += 32) {
            const uint32_t k = exit_out[ff + i] & 15u;
            const uint32_t c = class_id[ff + i];
            atomicAdd(&hist[k], 1u);
            if (c < 10) atomicAdd(&hist[16 + c * 16 + k], 1u);
        }
        if (lane == 0) {
            sg += best_gain[w];
            sc += best_cost[w];
            nw += 1;
            nf += N;
            ni += feasible[w] ? 0 : 1;
        }
    }
    if (lane == 0) {
        atomicAdd(&tot[0], (unsigned long long)sg);
        atomicAdd(&tot[1], (unsigned long long)sc);
        atomicAdd(&tot[2], (unsigned long long)nw);
        atomicAdd(&tot[3], (unsigned long long)nf);
        atomicAdd(&tot[4], (unsigned long long)ni);
    }
    __syncthreads();
    for (int x = threadIdx.x; x < 176; x += blockDim.x)
        if (hist[x]) atomicAdd(&stats[x], (unsigned long long)hist[x]);
    if (threadIdx.x < 5 && tot[threadIdx.x]) atomicAdd(&stats[176 + threadIdx.x], tot[threadIdx.x]);
}

cudaError_t launch_stats(const turbo_window_t *windows, int32_t num_windows, const uint8_t *class_id,
                         const uint8_t *exit_out, const int32_t *best_gain, const int32_t *best_cost,
                         const uint8_t *feasible, int64_t *stats, int num_sms, cudaStream_t stream)
{
    if (num_windows <= 0) return cudaSuccess;
    const int threads = 256;
    const int wpc = threads / 32;
    int64_t blocks = ((int64_t)num_windows + wpc - 1) / wpc;
    const int64_t cap = (int64_t)num_sms * 2;
    if (blocks > cap) blocks = cap;
    note_launch();
    stats_kernel<<<(unsigned)blocks, threads, 0, stream>>>(windows, num_windows, class_id, exit_out, best_gain,
                                                           best_cost, feasible,
                                                           reinterpret_cast<unsigned long long *>(stats));
    return cudaGetLastError();
}

}  // namespace turbo

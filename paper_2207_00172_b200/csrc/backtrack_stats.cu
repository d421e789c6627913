// backtrack_stats.cu -- K6 (plan reconstruction, a5) and K7 (plan statistics, a6).
#include "dp_kernel.cuh"

namespace turbo {

// ---------------------------------------------------------------------------------------------
// K6 (a5). Forward walk from (frame 0, b = C*): k_i = choice_i[b]; b -= c_{i,k_i}
// (the realisation of the lexicographic tie-break, reading R7; "we
// execute each frame according to the plan"). The chain of N dependent loads is latency-bound,
// so one warp serves one window and SPECULATES over the next D frames (backtrack_warp_spec in
// dp_kernel.cuh: every lane a candidate prefix, resolved by one ballot per round).
template <int K>
__device__ __noinline__ void backtrack_window(const uint32_t *__restrict__ gch, int32_t gtiles,
                                              const int32_t *__restrict__ oc, int32_t N, int32_t b,
                                              uint8_t *__restrict__ exit_g, int lane)
{
    auto cost = [&](int32_t i, int32_t k) -> int32_t { return __ldg(oc + (int64_t)i * K + k); };
    backtrack_warp_spec<K, DP_SOLVE_GLOBAL>(N, b, nullptr, gch, 0, gtiles, cost, exit_g, nullptr, lane);
}

__global__ void __launch_bounds__(128, 8) backtrack_kernel(const turbo_window_t *__restrict__ windows,
                                                        int32_t num_windows,
                                                        const int32_t *__restrict__ opt_cost,
                                                        const uint8_t *__restrict__ workspace,
                                                        const int32_t *__restrict__ best_cost,
                                                        const uint8_t *__restrict__ feasible,
                                                        uint8_t *__restrict__ exit_out)
{
    const int lane = threadIdx.x & 31;
    const int wpc = blockDim.x >> 5;
    for (int64_t w = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); w < num_windows;
         w += (int64_t)gridDim.x * wpc) {
        const int64_t ff = windows[w].first_frame;
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
        const int32_t *__restrict__ oc = opt_cost + windows[w].first_option;
        const int32_t b = best_cost[w];
        switch (K) {
#define TURBO_K_CASE(KK) \
    case KK: backtrack_window<KK>(gch, gtiles, oc, N, b, exit_out + ff, lane); break;
            TURBO_K_CASE(2) TURBO_K_CASE(3) TURBO_K_CASE(4) TURBO_K_CASE(5) TURBO_K_CASE(6)
            TURBO_K_CASE(7) TURBO_K_CASE(8) TURBO_K_CASE(9) TURBO_K_CASE(10) TURBO_K_CASE(11)
            TURBO_K_CASE(12) TURBO_K_CASE(13) TURBO_K_CASE(14) TURBO_K_CASE(15) TURBO_K_CASE(16)
#undef TURBO_K_CASE
            default: break;
        }
    }
}

cudaError_t launch_backtrack(const turbo_window_t *windows, int32_t num_windows, const int32_t *opt_cost,
                             const uint8_t *workspace, const int32_t *best_cost, const uint8_t *feasible,
                             uint8_t *exit_out, int num_sms, cudaStream_t stream)
{
    if (num_windows <= 0) return cudaSuccess;
    const int threads = 128;
    const int wpc = threads / 32;
    int64_t blocks = ((int64_t)num_windows + wpc - 1) / wpc;
    const int64_t cap = (int64_t)num_sms * 16;
    if (blocks > cap) blocks = cap;
    backtrack_kernel<<<(unsigned)blocks, threads, 0, stream>>>(windows, num_windows, opt_cost, workspace,
                                                               best_cost, feasible, exit_out);
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
    stats_kernel<<<(unsigned)blocks, threads, 0, stream>>>(windows, num_windows, class_id, exit_out, best_gain,
                                                           best_cost, feasible,
                                                           reinterpret_cast<unsigned long long *>(stats));
    return cudaGetLastError();
}

}  // namespace turbo

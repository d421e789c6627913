// next_steps.cu -- the steps just before and just after the hot path.
//
// NEXT-3 (before): the discriminator's difficulty score -> difficulty class (PAPER.md:511 buckets of
// width 0.1 on the training-time score; :525 theta'_x from D_f; reading R6: the class is the bucket
// of d = 1 - theta', clamped to [0, C-1]). HBM-bound: 4 B in, 1 B out per frame; float4 loads, one
// u32 (4 classes) store per thread. The integer decision is taken in IEEE float32 with explicit
// round-to-nearest intrinsics (no contraction), exactly as the oracle does.
//
// NEXT-2 (after): the plan -> per-exit batches ("organize the frames assigned by the
// same enhancement level to execute in a batch", :545): per window the batch sizes n_k, a stable
// partition of the window's frames by exit level, and (optionally) the executed latency
// f = sum_k I_k(n_k) of those batches. One warp per window; per 32-frame chunk and level, a ballot
// ranks the frames (arrival order preserved).
#include "turbo_internal.cuh"

namespace turbo {

__global__ void __launch_bounds__(256) bucketize_kernel(const float *__restrict__ theta, int64_t n, float inv_width,
                                                        int C, uint8_t *__restrict__ cls)
{
    const int64_t n4 = n >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n4; v += stride) {
        const float4 t = __ldcs(reinterpret_cast<const float4 *>(theta) + v);
        const uint32_t w = bucket_of(t.x, inv_width, C) | (bucket_of(t.y, inv_width, C) << 8) |
                           (bucket_of(t.z, inv_width, C) << 16) | (bucket_of(t.w, inv_width, C) << 24);
        __stcs(reinterpret_cast<uint32_t *>(cls) + v, w);
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
        const int64_t x = n4 * 4 + threadIdx.x;
        cls[x] = (uint8_t)bucket_of(theta[x], inv_width, C);
    }
}

cudaError_t launch_bucketize(const float *theta, int64_t n, int32_t C, float inv_width, uint8_t *cls, int num_sms,
                             cudaStream_t stream)
{
    if (n <= 0) return cudaSuccess;
    int64_t blocks = ((n >> 2) + 255) / 256;
    if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
    if (blocks < 1) blocks = 1;
    note_launch();
    bucketize_kernel<<<(unsigned)blocks, 256, 0, stream>>>(theta, n, inv_width, C, cls);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(256) batches_kernel(const turbo_window_t *__restrict__ windows, int32_t num_windows,
                                                      const uint8_t *__restrict__ exit_out, int32_t *__restrict__ count,
                                                      int32_t *__restrict__ order, const int32_t *__restrict__ batch,
                                                      int32_t cap, int64_t *__restrict__ latency,
                                                      int64_t *__restrict__ status)
{
    const int lane = threadIdx.x & 31;
    const int wpc = blockDim.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    for (int64_t w = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); w < num_windows;
         w += (int64_t)gridDim.x * wpc) {
        const int64_t ff = windows[w].first_frame;
        const int32_t N = windows[w].num_frames;
        // pass 1: batch sizes (lane k < 16 accumulates level k)
        int32_t mine = 0;
        for (int32_t i0 = 0; i0 < N; i0 += 32) {
            const int32_t i = i0 + lane;
            const uint32_t k = i < N ? exit_out[ff + i] : 0xffu;
            for (int kk = 0; kk < 16; ++kk) {
                const uint32_t m = __ballot_sync(0xffffffffu, k == (uint32_t)kk);
                if (lane == kk) mine += __popc(m);
            }
        }
        if (lane < 16) count[w * 16 + lane] = mine;
        if (latency != nullptr) {
            // executed latency f = sum_k I_k(n_k): lane k < K reads its level's table
            const int32_t K = windows[w].num_exits;
            const int64_t tab = (int64_t)windows[w].profile * 16 * (cap + 1);
            const bool over = lane < K && mine > cap;
            int64_t v = (lane < K && !over) ? (int64_t)batch[tab + (int64_t)lane * (cap + 1) + mine] : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            const bool bad = __any_sync(0xffffffffu, over);
            if (lane == 0) {
                latency[w] = bad ? -1 : v;
                if (bad) atomic_min_i64(&status[1], w);
            }
        }
        // exclusive prefix over levels -> base offset of each batch
        int32_t base = mine;
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int32_t u = __shfl_up_sync(0xffffffffu, base, o);
            if (lane >= o) base += u;
        }
        base -= mine;
        // pass 2: stable scatter (rank inside the chunk by ballot)
        for (int32_t i0 = 0; i0 < N; i0 += 32) {
            const int32_t i = i0 + lane;
            const uint32_t k = i < N ? exit_out[ff + i] : 0xffu;
            int32_t pos = 0;
            for (int kk = 0; kk < 16; ++kk) {
                const uint32_t m = __ballot_sync(0xffffffffu, k == (uint32_t)kk);
                const int32_t b = __shfl_sync(0xffffffffu, base, kk);
                if (k == (uint32_t)kk) pos = b + __popc(m & lt);
                if (lane == kk) base += __popc(m);
            }
            if (i < N) order[ff + pos] = i;
        }
    }
}

cudaError_t launch_batches(const turbo_window_t *windows, int32_t num_windows, const uint8_t *exit_out,
                           int32_t *count, int32_t *order, const int32_t *batch_cost, int32_t batch_cap,
                           int64_t *latency, int64_t *status, int num_sms, cudaStream_t stream)
{
    if (num_windows <= 0) return cudaSuccess;
    int64_t blocks = ((int64_t)num_windows + 7) / 8;
    if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
    note_launch();
    batches_kernel<<<(unsigned)blocks, 256, 0, stream>>>(windows, num_windows, exit_out, count, order, batch_cost,
                                                         batch_cap, latency, status);
    return cudaGetLastError();
}

}  // namespace turbo

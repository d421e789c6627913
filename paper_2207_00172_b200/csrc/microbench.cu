// microbench.cu -- the MEASURED shared-memory roofline denominator (bench.py).
//
// The DP kernels are bound by shared-memory bandwidth. MEASURED_PEAKS.json
// holds HBM and tensor-core peaks only, so the library carries its own smem stream kernel:
// every warp of every CTA issues conflict-free 32-bit shared loads (32 lanes x 4 B = one 128-B
// wavefront per instruction, the access type the DP uses), and the caller times the launch
// with CUDA events: peak = bytes / time. Not part of the method.
#include "turbo_internal.cuh"

namespace turbo {

constexpr int SMEM_BENCH_WORDS = 8192;           // 32 KB buffer per CTA
constexpr int SMEM_BENCH_THREADS = 1024;
constexpr int SMEM_BENCH_UNROLL = 32;

__global__ void __launch_bounds__(SMEM_BENCH_THREADS) smem_stream_kernel(int32_t iters, uint32_t *sink)
{
    __shared__ uint32_t buf[SMEM_BENCH_WORDS];
    for (int x = threadIdx.x; x < SMEM_BENCH_WORDS; x += blockDim.x) buf[x] = x * 2654435761u;
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(buf) + 4u * (threadIdx.x & 31);
    uint32_t row = (threadIdx.x >> 5) * 7u;           // warps start on different rows
    uint32_t acc = 0;
    for (int32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < SMEM_BENCH_UNROLL; ++u) {
            uint32_t v;
            const uint32_t addr = base + (((row + u) & (SMEM_BENCH_WORDS / 32 - 1)) << 7);
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
            acc += v;
        }
        row += SMEM_BENCH_UNROLL;
    }
    if (acc == 0x9e3779b9u) sink[threadIdx.x] = acc;  // keeps the loads; practically never stores
}

}  // namespace turbo

using namespace turbo;

extern "C" turbo_status_t turbo_debug_smem_stream(int32_t iters, int32_t ctas_per_sm, void *sink,
                                                  double *bytes_out, turbo_stream_t stream)
{
    if (iters < 1 || ctas_per_sm < 1 || ctas_per_sm > 2 || !sink || !bytes_out) return TURBO_ERR_INVALID_ARG;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TURBO_ERR_CUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return TURBO_ERR_CUDA;
    const int blocks = sms * ctas_per_sm;
    *bytes_out = (double)blocks * SMEM_BENCH_THREADS * (double)iters * SMEM_BENCH_UNROLL * 4.0;
    note_launch();
    smem_stream_kernel<<<blocks, SMEM_BENCH_THREADS, 0, (cudaStream_t)stream>>>(iters, (uint32_t *)sink);
    return cudaGetLastError() == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

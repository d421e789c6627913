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

// W = bytes per lane per load (4: ld.shared.u32, 8: .v2.u32, 16: .v4.u32); a warp instruction
// reads 32 W contiguous bytes = W / 4 wavefronts, conflict-free
template <int W>
__global__ void __launch_bounds__(SMEM_BENCH_THREADS) smem_stream_kernel(int32_t iters, uint32_t *sink)
{
    __shared__ uint32_t buf[SMEM_BENCH_WORDS];
    for (int x = threadIdx.x; x < SMEM_BENCH_WORDS; x += blockDim.x) buf[x] = x * 2654435761u;
    __syncthreads();
    constexpr uint32_t ROW = 32u * W;                 // bytes per warp instruction
    constexpr uint32_t ROWS = SMEM_BENCH_WORDS * 4u / ROW;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(buf) + (uint32_t)W * (threadIdx.x & 31);
    uint32_t row = (threadIdx.x >> 5) * 7u;           // warps start on different rows
    uint32_t acc = 0;
    for (int32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < SMEM_BENCH_UNROLL; ++u) {
            const uint32_t addr = base + ((row + u) & (ROWS - 1)) * ROW;
            if (W == 4) {
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
                acc += v;
            } else if (W == 8) {
                uint32_t a, b;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(addr));
                acc += a ^ b;
            } else {
                uint32_t a, b, c, d;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
                acc += (a ^ b) + (c ^ d);
            }
        }
        row += SMEM_BENCH_UNROLL;
    }
    if (acc == 0x9e3779b9u) sink[threadIdx.x] = acc;  // keeps the loads; practically never stores
}

}  // namespace turbo

using namespace turbo;

extern "C" turbo_status_t turbo_debug_smem_stream(int32_t iters, int32_t ctas_per_sm, int32_t bytes_per_lane,
                                                  void *sink, double *bytes_out, turbo_stream_t stream)
{
    if (iters < 1 || ctas_per_sm < 1 || ctas_per_sm > 2 || !sink || !bytes_out) return TURBO_ERR_INVALID_ARG;
    if (bytes_per_lane != 4 && bytes_per_lane != 8 && bytes_per_lane != 16) return TURBO_ERR_INVALID_ARG;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return TURBO_ERR_CUDA;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return TURBO_ERR_CUDA;
    const int blocks = sms * ctas_per_sm;
    *bytes_out = (double)blocks * SMEM_BENCH_THREADS * (double)iters * SMEM_BENCH_UNROLL * bytes_per_lane;
    note_launch();
    cudaStream_t st = (cudaStream_t)stream;
    if (bytes_per_lane == 4)
        smem_stream_kernel<4><<<blocks, SMEM_BENCH_THREADS, 0, st>>>(iters, (uint32_t *)sink);
    else if (bytes_per_lane == 8)
        smem_stream_kernel<8><<<blocks, SMEM_BENCH_THREADS, 0, st>>>(iters, (uint32_t *)sink);
    else
        smem_stream_kernel<16><<<blocks, SMEM_BENCH_THREADS, 0, st>>>(iters, (uint32_t *)sink);
    return cudaGetLastError() == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

// Self-test of the checked build's reporting path (tests/test_gpu_checked.py): one deliberately
// violated TCHECK -- a report in the checked library, nothing in the production one.
__global__ void tcheck_selftest_kernel(int32_t v)
{
    TCHECK(v != 7);
}

extern "C" turbo_status_t turbo_debug_tcheck_selftest(turbo_stream_t stream)
{
    note_launch();
    tcheck_selftest_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(7);
    return cudaGetLastError() == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

// copy.cu -- turbo_memcpy_sm: a copy done by the SMs instead of a copy engine (not a step of the
// method; the host <-> device transfer of a serving loop's per-step inputs and results). For the
// few tens of KB a scheduling step moves, a copy-engine transfer's fixed latency dominates; SMs
// reading (writing) mapped pinned host memory through UVA finish the same bytes sooner.
#include "turbo_internal.cuh"

namespace turbo {

constexpr int COPY_THREADS = 256;

__global__ void __launch_bounds__(COPY_THREADS) copy_sm_kernel(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src,
                                                            int64_t bytes, int vec)
{
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (vec) {                                            // both 16-B aligned: 16-B words, then the tail
        const int64_t n16 = bytes >> 4;
        const uint4 *s = reinterpret_cast<const uint4 *>(src);
        uint4 *d = reinterpret_cast<uint4 *>(dst);
        for (int64_t x = tid; x < n16; x += stride) d[x] = s[x];
        for (int64_t x = (n16 << 4) + tid; x < bytes; x += stride) dst[x] = src[x];
    } else {
        for (int64_t x = tid; x < bytes; x += stride) dst[x] = src[x];
    }
}

}  // namespace turbo

using namespace turbo;

extern "C" turbo_status_t turbo_memcpy_sm(void *dst, const void *src, size_t bytes, turbo_stream_t stream)
{
    if (bytes == 0) return TURBO_OK;
    if (!dst || !src) return TURBO_ERR_INVALID_ARG;
    const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
    const int64_t units = vec ? (int64_t)(bytes >> 4) : (int64_t)bytes;
    int64_t blocks = (units + COPY_THREADS - 1) / COPY_THREADS;
    blocks = blocks < 1 ? 1 : (blocks > 1184 ? 1184 : blocks);    // <= 8 CTAs per SM of 148
    note_launch();
    copy_sm_kernel<<<(unsigned)blocks, COPY_THREADS, 0, (cudaStream_t)stream>>>(
        static_cast<uint8_t *>(dst), static_cast<const uint8_t *>(src), (int64_t)bytes, vec ? 1 : 0);
    return cudaGetLastError() == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

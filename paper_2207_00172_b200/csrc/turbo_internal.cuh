// turbo_internal.cuh -- shared device helpers of the sm_100a kernels (product path).
// Nothing here is shared with oracle/ (the CPU oracle is independent by design).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "turbo.h"

// Checked build (TURBO_CHECKS=1 python -m paper_2207_00172_b200.build -> checked/libturbo.so): every
// TCHECK prints its location on a violated index bound instead of compiling to nothing.
// compute-sanitizer is closed on the GPU pool; tests/test_gpu_checked.py runs every kernel path of
// the checked library and fails on any report.
#ifdef TURBO_CHECKS
#include <cstdio>
#define TCHECK(cond)                                                                        \
    do {                                                                                    \
        if (!(cond))                                                                        \
            printf("TCHECK %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
                   (int)threadIdx.x, #cond);                                                \
    } while (0)
#else
#define TCHECK(cond) \
    do {             \
    } while (0)
#endif

namespace turbo {

// ---------------------------------------------------------------------------------------------
// Packed DP key: a row cell holds R = S << 4 (low 4 bits zero).
// Option k of a frame is pre-packed as gp_k = (g_k << 4) | (15 - k), so the max-plus update
//   key = max_k (R_old[b - c_k] + gp_k)
// carries the argmax in its low 4 bits; equal S prefer the larger tag = the SMALLER k, which
// is the per-cell tie-break that realises the lexicographic order (reading R7).
//   R_new = key & ~15,   choice = 15 - (key & 15) = (key & 15) ^ 15.
// -inf: NEG_R = -2^30. With the range rule sum_i max_k |g_ik| < 2^25 every reachable value of
// a feasible cell lies in (-2^29, 2^29) and every infeasible one in (-1.5*2^30, -2^29), so the
// two bands never mix and nothing overflows int32 (reading R14).
constexpr int32_t NEG_R = -(1 << 30);
constexpr int32_t VALID_MIN_R = -(1 << 29);     // feasible  <=>  R > VALID_MIN_R
constexpr int64_t GAIN_RANGE_LIMIT = (int64_t)1 << 25;
constexpr int MAX_EXITS = 16;

__host__ __device__ __forceinline__ int choice_bits(int K) { return K <= 4 ? 2 : 4; }
// rows of 32 cells per choice word (= per tile): 16 for 2-bit, 8 for 4-bit choices
__host__ __device__ __forceinline__ int rows_per_tile(int K) { return 32 / choice_bits(K); }
// row-size class of a window with `cells` = budget_bound + 1 (TURBO_NUM_CLASSES = long window)
__host__ __device__ __forceinline__ int row_class(int64_t cells)
{
    return cells <= TURBO_CLASS_CELLS_0 ? 0 : cells <= TURBO_CLASS_CELLS_1 ? 1 : cells <= TURBO_CLASS_CELLS_2 ? 2
         : cells <= TURBO_CLASS_CELLS_3 ? 3 : TURBO_NUM_CLASSES;
}

__host__ __device__ __forceinline__ int64_t num_rows(int64_t B) { return (B + 1 + 31) / 32; }
__host__ __device__ __forceinline__ int64_t num_tiles(int64_t B, int K) {
    int64_t rpt = rows_per_tile(K);
    return (num_rows(B) + rpt - 1) / rpt;
}
// bytes of one window's choice plane: N frames x tiles x 32 lanes x 4 B
__host__ __device__ __forceinline__ int64_t choice_plane_bytes(int64_t N, int64_t B, int K) {
    return N * num_tiles(B, K) * 128;
}

// bit offset of row j's choice field inside its tile word (see pack_choices in dp_kernel.cuh)
__host__ __device__ __forceinline__ int choice_shift(int j, int CB) { return 8 * (j & 3) + CB * (j >> 2); }

__device__ __forceinline__ int32_t max_plus(int32_t a, int32_t b, int32_t c) {
    return __viaddmax_s32(a, b, c);          // max(a + b, c): one VIADDMNMX on sm_90+/sm_100a
}

__device__ __forceinline__ void atomic_min_i64(int64_t *p, int64_t v) {
    // status words use -1 (all ones) as "none": an unsigned min keeps the smallest index
    atomicMin(reinterpret_cast<unsigned long long *>(p), (unsigned long long)v);
}


// ---------------------------------------------------------------------------------------------
// DP launch parameters (dp_warp.cu) and the host-side launchers of every kernel.
enum DpMode { DP_PLAN = 0, DP_SOLVE_SMEM = 1, DP_SOLVE_GLOBAL = 2 };

struct DpParams {
    const turbo_window_t *windows;
    int32_t num_windows;
    int32_t row_words;      // per-warp row capacity (multiple of 32)
    int32_t chs_words;      // per-warp smem choice capacity (DP_SOLVE_SMEM)
    int32_t cst_words;      // smem words after the rows: option table (osm) or costs (solve)
    int32_t warp_words;     // unused (0)
    int32_t pad_words;      // -inf words below each row buffer (unchecked shifts up to this)
    int32_t osm;            // 1: options staged in smem (cst_words = 2 * frames * exits)
    int32_t warps_per_cta;
    const int32_t *opt_gain;
    const int32_t *opt_cost;
    uint8_t *workspace;
    int32_t *best_gain;
    int32_t *best_cost;
    uint8_t *feasible;
    uint8_t *exit_out;
    int64_t *status;
    // turbo_schedule (fused a1..a6) only
    const turbo_profile_t *profiles;
    turbo_window_t *windows_rw;
    const uint8_t *class_id;
    const int32_t *capacity;
    int32_t base_cost;
    int32_t fuse;
    int32_t max_options;    // option-table entries per window (osm); fused scratch follows it
    int32_t prof_entries;   // fused: staged profile entries (max C*K)
    int64_t grid_scratch_offset;   // long-window kernel: workspace offset of flags + halo ring
    int32_t debug;                 // long-window kernel tuning switches (TURBO_GRID_DEBUG)
    int32_t cls;                   // row-size class served by this launch (-1: every window)
    int32_t cls_count;             // windows in that class (residency / wave planning)
    int32_t ordered;               // serve windows[cls_first + r].order, r < cls_count (LPT order)
    int32_t cls_first;
    int64_t *stats;
    int64_t *trace;                // debug: per-CTA phase timestamps (turbo_debug_trace)
    int64_t trace_words;
    // lockstep kernel (dp_pack.cu): windows per CTA, tiles per window, words per window slot
    int32_t max_frames;
    int32_t pack_v;
    int32_t pack_tiles;
    int32_t pack_stride;
    int32_t generic;               // mixed-K plan-mode launch: the runtime-K kernel (dp_gen.cu)
    int32_t grid_max_budget;       // long-window kernel: largest budget bound (L2-row path row size)
    // turbo_schedule_theta (NEXT-3 fused): classes from the difficulty scores, written to class_out
    const float *theta;
    float inv_width;
    uint8_t *class_out;
    int32_t u16;                   // NEXT-5: u16 rows for the windows that qualify (opt-in: variant bit 128)
    int64_t *u16_count;            // test hook (turbo_debug_u16_counter): windows planned on u16 rows
    int32_t small;                 // <= 4-warp launches may use the 72-register kernels (variant bit 256 clears)
    int32_t cluster_cap;           // long rows up to this many cells take the cluster kernel (0: none)
};

// NEXT-3 (PAPER.md:511 buckets of width 0.1; :525 theta'_x from D_f; reading R6): the class of a
// difficulty score = the bucket of d = 1 - theta, clamped to [0, C-1], decided in IEEE float32 with
// explicit round-to-nearest operations (no contraction); NaN -> class 0.
__device__ __forceinline__ uint32_t bucket_of(float theta, float inv_width, int C)
{
    const float d = __fsub_rn(1.0f, theta);
    const float q = __fmul_rn(d, inv_width);
    int c = 0;
    if (q >= (float)C)
        c = C - 1;
    else if (q >= 0.0f)
        c = (int)floorf(q);                          // NaN fails both tests -> class 0
    return (uint32_t)min(c, C - 1);
}

// The class of frame idx of a fused launch (turbo_schedule: the class-id input; turbo_schedule_theta:
// the bucket of its score under the window's profile's C classes)
__device__ __forceinline__ int32_t frame_class(const DpParams &P, int64_t idx, int32_t C)
{
    if (P.theta != nullptr) return (int32_t)bucket_of(__ldg(P.theta + idx), P.inv_width, C);
    return (int32_t)P.class_id[idx];
}

// turbo_debug_trace: %globaltimer at phase p of window w (thread 0 of the window's CTA). Compiled
// in only with -DTURBO_TRACE (TURBO_TRACE=1 python -m paper_2207_00172_b200.build): the marks
// change the register allocation of the 64-register DP kernels, so production builds omit them.
__device__ __forceinline__ void trace_mark(const DpParams &P, int64_t w, int p)
{
#ifdef TURBO_TRACE
    if (P.trace != nullptr && threadIdx.x == 0 && w * 8 + 8 <= P.trace_words) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.trace[w * 8 + p] = (int64_t)t;
    }
#endif
}

// Does pick_dp_kernel use a fixed-K kernel (K in {4, 5, 6, 8} for every window of the launch)?
// Fixed-K kernels serve windows in index order; the mixed-K kernel follows the serving order.
__host__ __device__ inline bool dp_kernel_fixed_k(int kmin, int kmax)
{
    return kmin == kmax && (kmin == 4 || kmin == 5 || kmin == 6 || kmin == 8);
}

cudaError_t launch_batched(const turbo_window_t *windows, int32_t num_windows, const turbo_profile_t *profiles,
                           const int32_t *batch, int32_t cap, const uint8_t *class_id, int32_t *best_gain,
                           int32_t *best_cost, uint8_t *feasible, uint8_t *exit_out, int64_t *status, int32_t kmax,
                           int32_t max_frames, void *workspace, int32_t general, int num_sms, cudaStream_t stream);
int64_t batched_dp_bytes(int32_t max_frames, int32_t max_exits, int num_sms);
// every kernel launch of the library is counted (turbo_launch_count)
void note_launch();

struct DpLaunch {
    int mode;
    int warps_per_cta;
    int blocks;
    size_t smem_bytes;
};

cudaError_t launch_lookup(const turbo_profile_t *profiles, turbo_window_t *windows, int32_t num_windows,
                          const uint8_t *class_id, const int32_t *capacity, int32_t base_cost, int32_t *opt_gain,
                          int32_t *opt_cost, int64_t *status, int32_t max_options, int num_sms, cudaStream_t stream);
cudaError_t launch_dp(const turbo_shape_t *shape, int mode, const DpParams &P, int num_sms, int smem_per_sm,
                      int smem_per_cta_max, cudaStream_t stream, DpLaunch *info);
int dp_warps_per_window(const turbo_shape_t *shape);
// host-only validation (no launch): the class kernel fits its shared memory / the long-window
// kernel fits shared memory and the cooperative grid fits the device
cudaError_t check_dp(const turbo_shape_t *shape, int mode, const DpParams &P, int smem_per_cta_max);
cudaError_t check_dp_grid(const turbo_shape_t *shape, int mode, int num_sms, int smem_per_cta_max, int32_t cluster_cap);

// long-window (grid) kernel: scratch = flags (pub/con per CTA + misc) + halo ring
constexpr int GRID_MAX_CTAS = 512;                 // two CTAs per SM on 148 SMs
constexpr int GRID_H = TURBO_BIG_MAX_COST;         // halo capacity of the segment path (cells)
constexpr int GRID_THREADS = 512;                  // threads per CTA of the long-window DP kernel
constexpr int GRID_CTAS_PER_SM = 1;                // (2 x 256 threads measured slower on c4: 7.1 vs 5.9 ms)
constexpr int GRID_RING_DEPTH = 8;
// scratch = [flags: cleared by every launch][header: persists across launches][halo ring]
__host__ __device__ constexpr int64_t grid_flags_words() { return 2 * GRID_MAX_CTAS + 64 + 16 * GRID_MAX_CTAS; }
// header (64 B): {magic u64, tag epoch i32}. The ring's step tags continue from the epoch stored in the
// workspace itself, so tags never repeat within a workspace -- also across CUDA-graph replays, whose
// kernel arguments are frozen at capture (the kernel advances the epoch on the device).
constexpr int64_t GRID_HEADER_WORDS = 16;
constexpr unsigned long long GRID_MAGIC = 0x7475726230677264ull;   // "turb0grd"
__host__ __device__ constexpr int64_t grid_ring_words() { return (int64_t)GRID_RING_DEPTH * GRID_MAX_CTAS * GRID_H; }
// cells of one global row of the L2-row path: whole 512-cell tiles above the largest budget
__host__ __device__ constexpr int64_t grid_l2_stride(int64_t max_budget) { return (max_budget + 1 + 511) & ~(int64_t)511; }
// scratch = [flags][header][halo ring: 8-B words][two global rows (L2-row path): int32]
__host__ __device__ constexpr int64_t grid_scratch_bytes(int64_t max_budget)
{
    return 4 * (grid_flags_words() + GRID_HEADER_WORDS) + 8 * grid_ring_words() + 8 * grid_l2_stride(max_budget);
}
cudaError_t launch_heuristic(const turbo_shape_t *shape, const turbo_window_t *windows, const int32_t *opt_gain,
                             const int32_t *opt_cost, int32_t *gain_out, int32_t *cost_out, uint8_t *feasible,
                             uint8_t *exit_out, int32_t *steps, int num_sms, int smem_per_cta_max,
                             cudaStream_t stream);
cudaError_t launch_bucketize(const float *theta, int64_t n, int32_t C, float inv_width, uint8_t *cls, int num_sms,
                             cudaStream_t stream);
cudaError_t launch_batches(const turbo_window_t *windows, int32_t num_windows, const uint8_t *exit_out,
                           int32_t *count, int32_t *order, const int32_t *batch_cost, int32_t batch_cap,
                           int64_t *latency, int64_t *status, int num_sms, cudaStream_t stream);
// lockstep multi-window kernel for short-row single-class batches (dp_pack.cu)
bool pack_geometry(const turbo_shape_t *s, const DpParams &P, int num_sms, int smem_per_cta_max, int *V_out,
                   int *T_out, int *warps_out, size_t *smem_out);
cudaError_t launch_pack(const turbo_shape_t *s, const DpParams &P, int num_sms, int smem_per_cta_max,
                        cudaStream_t stream);
cudaError_t launch_dp_grid(const turbo_shape_t *shape, int mode, const DpParams &P, int num_sms,
                           int smem_per_cta_max, cudaStream_t stream);
// cluster kernel for long rows up to TURBO_CLUSTER_CELLS cells (dp_cluster.cu)
struct ClusterLaunch {
    const void *kern;
    int cs;                 // CTAs per cluster
    int32_t seg, lg_seg;    // cells per CTA segment (a power of two) and its log2
    size_t smem;
    int max_clusters;       // resident clusters on the device
};
cudaError_t cluster_geometry(const turbo_shape_t *shape, int smem_per_cta_max, ClusterLaunch *out);
cudaError_t launch_dp_cluster(const turbo_shape_t *shape, const DpParams &P, int smem_per_cta_max,
                              cudaStream_t stream);
size_t dp_smem_bytes(const DpParams &P, int nwarps);
// cls >= 0: only the windows of that row-size class (the others were walked elsewhere)
// Window selection of a per-class launch: the class's range of the serving order (ordered), or
// every window filtered by class (cls < 0: all windows).
struct WinSel {
    int32_t cls = -1;
    int32_t ordered = 0;
    int32_t first = 0;
    int32_t count = 0;
    __host__ __device__ int64_t n_iter(int64_t W) const { return ordered ? count : W; }
    // window of iteration r, or -1 when the class filter skips it
    __device__ __forceinline__ int64_t window(const turbo_window_t *windows, int64_t r) const
    {
        if (ordered) return windows[first + r].order;
        if (cls >= 0 && row_class((int64_t)windows[r].budget_bound + 1) != cls) return -1;
        return r;
    }
};
cudaError_t launch_backtrack(const turbo_window_t *windows, int32_t num_windows, const int32_t *opt_cost,
                             const uint8_t *workspace, const int32_t *best_cost, const uint8_t *feasible,
                             uint8_t *exit_out, int num_sms, cudaStream_t stream, WinSel sel = WinSel());
// turbo_schedule, windows of row-size class cls whose DP ran in plan mode: a5 walk with costs from
// class ids + profile, then a6 statistics of those windows
cudaError_t launch_walk_sched(const turbo_window_t *windows, int32_t num_windows, const turbo_profile_t *profiles,
                              const uint8_t *class_id, const uint8_t *workspace, const int32_t *best_gain,
                              const int32_t *best_cost, const uint8_t *feasible, uint8_t *exit_out, int64_t *stats,
                              int num_sms, cudaStream_t stream, WinSel sel);
cudaError_t launch_stats(const turbo_window_t *windows, int32_t num_windows, const uint8_t *class_id,
                         const uint8_t *exit_out, const int32_t *best_gain, const int32_t *best_cost,
                         const uint8_t *feasible, int64_t *stats, int num_sms, cudaStream_t stream);

}  // namespace turbo

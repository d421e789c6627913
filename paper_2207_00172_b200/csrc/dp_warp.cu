// dp_warp.cu -- K2/K5 (+ fused K6): the MCKP max-plus DP, one warp per window.
//
// Method (§5.2, with f = sum, reading R1; exact = the paper's "upper",
// PAPER.md:858 §6.4). Frames are processed in REVERSE (i = N-1 .. 0) so that the forward
// backtrack realises the lexicographic tie-break with frame 0 most significant (reading R7):
//     S_N[b] = 0,   S_i[b] = max_{k : c_ik <= b} ( g_ik + S_{i+1}[b - c_ik] ),   b = 0..B
//     choice_i[b] = smallest maximising k;  G* = S_0[B];  C* = #{b <= B : S_0[b] < G*}
// (S_0 is non-decreasing in b, so the count is the first b reaching G*).
//
// B200 mapping:
//  * the budget row lives in shared memory, ONE buffer per window, updated IN PLACE tile by
//    tile from the top (b large) down: a cell only ever reads cells <= itself (c >= 0), so
//    a tile's reads never touch the (already updated) tiles above it;
//  * cell b = row*32 + lane: for a warp-uniform shift c the 32 lanes read 32 consecutive
//    words -> conflict-free LDS; one VIADDMNMX (add + max) per option per cell;
//  * argmax rides in the low 4 bits of the packed key (turbo_internal.cuh);
//  * choices are packed 8 (4-bit) or 16 (2-bit) rows per u32 -> one coalesced 128-B store
//    per warp per tile, to HBM (plan) or to shared memory (fused solve, when it fits);
//  * per frame, lane k < K holds option k in a register (loaded one frame ahead) and the
//    warp broadcasts them with shuffles; no block barrier anywhere (only __syncwarp).
#include "turbo_internal.cuh"

namespace turbo {

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int K, int MODE>
__device__ __forceinline__ void dp_window(const DpParams &P, int64_t w, int32_t *__restrict__ row,
                                          uint32_t *__restrict__ sch, int32_t *__restrict__ cst, int lane)
{
    constexpr int CB = (K <= 4) ? 2 : 4;          // choice bits
    constexpr int RPT = 32 / CB;                   // rows of 32 cells per tile (per choice word)
    constexpr uint32_t CMASK = (1u << CB) - 1u;

    const turbo_window_t *win = P.windows + w;
    const int64_t ff = win->first_frame;
    const int64_t fo = win->first_option;
    const int32_t N = win->num_frames;
    const int32_t B = win->budget;
    const int32_t Bb = win->budget_bound;
    const int64_t choff = win->choice_offset;

    const int32_t *__restrict__ og = P.opt_gain + fo;
    const int32_t *__restrict__ oc = P.opt_cost + fo;

    // ---- prologue: validation + sums for the infeasible report (reading R8)
    int64_t abs_sum = 0, g0_sum = 0, c0_sum = 0;
    bool bad = (B < 0) || (B > Bb);
    for (int32_t i = lane; i < N; i += 32) {
        int32_t m = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int32_t g = __ldg(og + (int64_t)i * K + k);
            const int32_t c = __ldg(oc + (int64_t)i * K + k);
            const int32_t a = g < 0 ? -g : g;
            m = a > m ? a : m;
            bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
            if (k == 0) {
                g0_sum += g;
                c0_sum += c;
            }
        }
        abs_sum += m;
    }
    abs_sum = warp_sum_i64(abs_sum);
    g0_sum = warp_sum_i64(g0_sum);
    c0_sum = warp_sum_i64(c0_sum);
    bad = __any_sync(0xffffffffu, bad) || abs_sum >= GAIN_RANGE_LIMIT || c0_sum >= 0x7fffffffll;

    if (bad) {
        if (lane == 0) {
            P.best_gain[w] = 0;
            P.best_cost[w] = 0;
            P.feasible[w] = 0;
            atomic_min_i64(&P.status[1], w);
        }
        if (MODE != DP_PLAN)
            for (int32_t i = lane; i < N; i += 32) P.exit_out[ff + i] = 0;
        return;
    }

    const int32_t nrows = (B + 32) >> 5;
    const int32_t ntiles = (nrows + RPT - 1) / RPT;
    // choice-plane stride (tiles per frame): the layout bound for global planes, exact for smem
    const int32_t gtiles = (int32_t)(((Bb + 32) >> 5) + RPT - 1) / RPT;
    uint32_t *__restrict__ gch = reinterpret_cast<uint32_t *>(P.workspace + choff);

    // S_N = 0 on every cell (including the padding cells above B in the last row)
    for (int32_t x = lane; x < nrows * 32; x += 32) row[x] = 0;

    // options of frame i live in lane k < K: packed gain (g << 4 | 15 - k) and cost
    int32_t my_gp = 0, my_c = 0;
    if (N > 0 && lane < K) {
        my_gp = (__ldg(og + (int64_t)(N - 1) * K + lane) << 4) | (15 - lane);
        my_c = __ldg(oc + (int64_t)(N - 1) * K + lane);
    }
    __syncwarp();

    for (int32_t i = N - 1; i >= 0; --i) {
        int32_t gp[K], cc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            gp[k] = __shfl_sync(0xffffffffu, my_gp, k);
            cc[k] = __shfl_sync(0xffffffffu, my_c, k);
        }
        if (MODE != DP_PLAN && lane < K) cst[i * K + lane] = my_c;
        if (i > 0 && lane < K) {                       // prefetch frame i-1
            my_gp = (__ldg(og + (int64_t)(i - 1) * K + lane) << 4) | (15 - lane);
            my_c = __ldg(oc + (int64_t)(i - 1) * K + lane);
        }
        for (int32_t t = ntiles - 1; t >= 0; --t) {
            const int32_t row0 = t * RPT;
            const int32_t nr = min(RPT, nrows - row0);
            const int32_t b_lo = row0 * 32;
            const int32_t b_hi = b_lo + nr * 32 - 1;
            int32_t key[RPT];
#pragma unroll
            for (int r = 0; r < RPT; ++r) key[r] = NEG_R;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int32_t c = cc[k];
                const int32_t g = gp[k];
                if (c <= b_lo) {                              // every cell of the tile can take k
                    const int32_t *__restrict__ src = row + (b_lo + lane - c);
#pragma unroll
                    for (int r = 0; r < RPT; ++r)
                        if (r < nr) key[r] = max_plus(src[r * 32], g, key[r]);
                } else if (c <= b_hi) {                       // low cells: b < c reads -inf
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        if (r < nr) {
                            const int32_t idx = b_lo + r * 32 + lane - c;
                            int32_t v = row[idx < 0 ? 0 : idx];
                            v = idx < 0 ? NEG_R : v;
                            key[r] = max_plus(v, g, key[r]);
                        }
                    }
                }
            }
            __syncwarp();                                     // all reads of this tile done
            uint32_t word = 0;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                if (r < nr) {
                    row[b_lo + r * 32 + lane] = key[r] & ~15;
                    word |= ((uint32_t)key[r] & CMASK) << (CB * r);
                }
            }
            word ^= 0xffffffffu;                              // tag (15 - k) -> k per field
            if (MODE == DP_SOLVE_SMEM)
                sch[(i * ntiles + t) * 32 + lane] = word;
            else
                gch[((int64_t)i * gtiles + t) * 32 + lane] = word;
        }
        __syncwarp();                                         // frame i visible to frame i-1
    }

    // ---- a4: optimum extraction
    const int32_t RB = row[B];
    const bool feas = RB > VALID_MIN_R;
    int32_t cnt = 0;
    for (int32_t b = lane; b <= B; b += 32) cnt += row[b] < RB ? 1 : 0;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    const int32_t G = feas ? (RB >> 4) : (int32_t)g0_sum;
    const int32_t Cst = feas ? cnt : (int32_t)c0_sum;
    if (lane == 0) {
        P.best_gain[w] = G;
        P.best_cost[w] = Cst;
        P.feasible[w] = feas ? 1 : 0;
    }
    if (MODE == DP_PLAN) return;

    // ---- a5 fused: forward backtrack from (frame 0, b = C*)
    if (!feas) {
        for (int32_t i = lane; i < N; i += 32) P.exit_out[ff + i] = 0;
        return;
    }
    __syncwarp();
    if (lane == 0) {
        int32_t b = Cst;
        for (int32_t i = 0; i < N; ++i) {
            const int32_t t = b / (32 * RPT);
            const int32_t j = (b >> 5) & (RPT - 1);
            uint32_t word;
            if (MODE == DP_SOLVE_SMEM)
                word = sch[(i * ntiles + t) * 32 + (b & 31)];
            else
                word = gch[((int64_t)i * gtiles + t) * 32 + (b & 31)];
            const int32_t k = (int32_t)((word >> (CB * j)) & CMASK);
            P.exit_out[ff + i] = (uint8_t)k;
            b -= cst[i * K + k];
        }
    }
}

template <int KSEL, int MODE>
__global__ void __launch_bounds__(128) dp_warp_kernel(DpParams P)
{
    extern __shared__ int4 smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    int32_t *base = reinterpret_cast<int32_t *>(smem_raw) + (int64_t)warp * P.warp_words;
    int32_t *row = base;
    uint32_t *sch = reinterpret_cast<uint32_t *>(base + P.row_words);
    int32_t *cst = base + P.row_words + P.chs_words;
    for (int64_t w = (int64_t)blockIdx.x * P.warps_per_cta + warp; w < P.num_windows;
         w += (int64_t)gridDim.x * P.warps_per_cta) {
        if (KSEL != 0) {
            dp_window<(KSEL > 0 ? KSEL : 2), MODE>(P, w, row, sch, cst, lane);
        } else {
            switch (P.windows[w].num_exits) {
#define TURBO_K_CASE(KK) case KK: dp_window<KK, MODE>(P, w, row, sch, cst, lane); break;
                TURBO_K_CASE(2) TURBO_K_CASE(3) TURBO_K_CASE(4) TURBO_K_CASE(5) TURBO_K_CASE(6)
                TURBO_K_CASE(7) TURBO_K_CASE(8) TURBO_K_CASE(9) TURBO_K_CASE(10) TURBO_K_CASE(11)
                TURBO_K_CASE(12) TURBO_K_CASE(13) TURBO_K_CASE(14) TURBO_K_CASE(15) TURBO_K_CASE(16)
#undef TURBO_K_CASE
                default: break;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
typedef void (*dp_kernel_t)(DpParams);

template <int MODE>
static dp_kernel_t pick_kernel(int kmin, int kmax)
{
    if (kmin != kmax) return dp_warp_kernel<0, MODE>;
    switch (kmin) {
#define TURBO_K_PICK(KK) case KK: return dp_warp_kernel<KK, MODE>;
        TURBO_K_PICK(2) TURBO_K_PICK(3) TURBO_K_PICK(4) TURBO_K_PICK(5) TURBO_K_PICK(6)
        TURBO_K_PICK(7) TURBO_K_PICK(8) TURBO_K_PICK(9) TURBO_K_PICK(10) TURBO_K_PICK(11)
        TURBO_K_PICK(12) TURBO_K_PICK(13) TURBO_K_PICK(14) TURBO_K_PICK(15) TURBO_K_PICK(16)
#undef TURBO_K_PICK
        default: return dp_warp_kernel<0, MODE>;
    }
}

// Choose the per-SM concurrency s (windows resident per SM) minimising
// ceil(W / (num_sms * s)) * s -- equal-size windows finish in waves, so the tail wave is the
// quantisation loss -- among the s the shared memory allows; ties go to the larger s.
static int pick_concurrency(int64_t W, int num_sms, int s_max)
{
    int best_s = 1;
    int64_t best_cost = INT64_MAX;
    for (int s = 1; s <= s_max; ++s) {
        int64_t slots = (int64_t)num_sms * s;
        int64_t cost = ((W + slots - 1) / slots) * s;
        if (cost < best_cost || (cost == best_cost && s > best_s)) {
            best_cost = cost;
            best_s = s;
        }
    }
    return best_s;
}

cudaError_t launch_dp(const turbo_shape_t *shape, int mode, const DpParams &P0, int num_sms, int smem_per_sm,
                      int smem_per_cta_max, cudaStream_t stream, DpLaunch *info)
{
    DpParams P = P0;
    const int64_t W = shape->num_windows;
    if (W <= 0) return cudaSuccess;
    // one warp per CTA: the block scheduler then balances windows per SM at warp granularity
    const int wpc = 1;
    P.warps_per_cta = wpc;
    const size_t bytes_per_warp = (size_t)P.warp_words * 4;
    const size_t reserve = 1024;                      // per-CTA system reservation on sm_100
    int s_max = (int)(smem_per_sm / (bytes_per_warp * wpc + reserve));
    if (s_max > 32) s_max = 32;                       // max resident CTAs per SM
    if (s_max < 1) return cudaErrorInvalidConfiguration;
    int s = pick_concurrency(W, num_sms, s_max);
    // pad the dynamic smem so that exactly s CTAs fit per SM (occupancy as a knob)
    size_t smem = bytes_per_warp * wpc;
    size_t padded = smem_per_sm / s - reserve;
    if (padded > (size_t)smem_per_cta_max) padded = smem_per_cta_max;
    if (padded > smem) smem = padded & ~(size_t)15;
    int blocks = (int)((W + wpc - 1) / wpc);
    dp_kernel_t kern = (mode == DP_PLAN)          ? pick_kernel<DP_PLAN>(shape->min_exits, shape->max_exits)
                       : (mode == DP_SOLVE_SMEM) ? pick_kernel<DP_SOLVE_SMEM>(shape->min_exits, shape->max_exits)
                                                 : pick_kernel<DP_SOLVE_GLOBAL>(shape->min_exits, shape->max_exits);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<blocks, 32 * wpc, smem, stream>>>(P);
    if (info) {
        info->mode = mode;
        info->warps_per_cta = wpc;
        info->blocks = blocks;
        info->smem_bytes = smem;
    }
    return cudaGetLastError();
}

}  // namespace turbo

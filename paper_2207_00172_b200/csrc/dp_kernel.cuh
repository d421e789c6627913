// dp_kernel.cuh -- K2/K3/K5 (+ fused K6): the MCKP max-plus DP, one CTA of G warps per window.
//
// Method (§5.2, with f = sum, reading R1; exact = the paper's "upper",
// PAPER.md:858 §6.4). Frames are processed in REVERSE (i = N-1 .. 0) so that the forward
// backtrack realises the lexicographic tie-break with frame 0 most significant (reading R7):
//     S_N[b] = 0,   S_i[b] = max_{k : c_ik <= b} ( g_ik + S_{i+1}[b - c_ik] ),   b = 0..B
//     choice_i[b] = smallest maximising k;  G* = S_0[B];  C* = #{b <= B : S_0[b] < G*}
// (S_0 is non-decreasing in b, so the count is the first b reaching G*).
//
// B200 mapping:
//  * the budget row lives in shared memory; cell b = row*32 + lane, so for a warp-uniform shift
//    c the 32 lanes read 32 consecutive words (conflict-free LDS) and one VIADDMNMX (add+max)
//    does one option of one cell; the argmax rides in the low 4 bits of the packed key;
//  * a tile = 8 (4-bit choices) or 16 (2-bit) rows of 32 cells: each lane packs its tile's
//    choices into one u32 -> one coalesced 128-B store per warp per tile, to HBM (plan) or to
//    shared memory (fused solve, when the window's planes fit);
//  * G = 1 warp: ONE row buffer updated IN PLACE tile by tile from the top down (a cell only
//    reads cells <= itself) with only __syncwarp; G > 1 warps: tiles t = warp, warp+G, ...,
//    rows double-buffered, one CTA barrier per frame;
//  * per frame, lane k < K of every warp holds option k (prefetched one frame ahead) and the
//    warp broadcasts it with shuffles.
#pragma once

#include <type_traits>

#include "turbo_internal.cuh"

namespace turbo {

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// a4's C* = min{b <= B : S_0[b] = G*} by ONE warp: S_0 is non-decreasing in b over the feasible
// cells and every infeasible cell (a prefix of the row) lies below any feasible value (R14), so
// "S_0[b] >= S_0[B]" is false ... false, true ... true on [0, B] and a 32-ary search finds its first
// true cell in ceil(log_31(B + 1)) + 1 rounds of one load and one vote (B = 1000: 3 rounds) --
// instead of counting the B + 1 cells below G* with every thread and a CTA-wide reduction.
// (T = int32_t: packed-key rows; T = uint16_t: the u16 rows of NEXT-5, values S + V0)
template <class T>
__device__ __forceinline__ int32_t warp_first_at_least(const T *__restrict__ S, int32_t B, int32_t RB, int lane)
{
    int32_t lo = 0, hi = B;                               // invariant: answer in [lo, hi], S[hi] >= RB
    while (hi - lo >= 32) {
        const int32_t step = (hi - lo + 30) / 31;         // lane 31 probes >= hi
        const int32_t p = min(lo + lane * step, hi);
        const unsigned m = __ballot_sync(0xffffffffu, (int32_t)S[p] >= RB);
        const int f = __ffs(m) - 1;                       // m != 0: lane 31 probes hi
        const int32_t nhi = min(lo + f * step, hi);
        lo = f == 0 ? lo : lo + (f - 1) * step + 1;
        hi = nhi;
    }
    const int32_t p = lo + lane;
    const unsigned m = __ballot_sync(0xffffffffu, p > hi || (int32_t)S[min(p, hi)] >= RB);
    return lo + __ffs(m) - 1;
}

// One tile of one frame: keys of RPT rows (cells b_lo + r*32 + lane) from row `src`.
// `src` is preceded by `pad` words of -inf, so an option whose shift stays inside the pad
// (c <= b_lo + pad) needs no bounds check; only larger shifts in the lowest tiles take the
// predicated path (cells b < c read -inf).
template <int K, int RPT>
__device__ __forceinline__ void tile_keys(const int32_t *__restrict__ src, int32_t b_lo, int32_t nr, int32_t pad,
                                          const int32_t (&gp)[K], const int32_t (&cc)[K], int lane,
                                          int32_t (&key)[RPT])
{
    const int32_t b_hi = b_lo + nr * 32 - 1;
#pragma unroll
    for (int r = 0; r < RPT; ++r) key[r] = NEG_R;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int32_t c = cc[k];
        const int32_t g = gp[k];
        if (c <= b_lo + pad) {                                // unchecked: shifts stay in the pad
            const int32_t *__restrict__ s = src + (b_lo + lane - c);
            if (nr == RPT) {
#pragma unroll
                for (int r = 0; r < RPT; ++r) key[r] = max_plus(s[r * 32], g, key[r]);
            } else {
#pragma unroll
                for (int r = 0; r < RPT; ++r)
                    if (r < nr) key[r] = max_plus(s[r * 32], g, key[r]);
            }
        } else if (c <= b_hi) {                               // low cells: b < c reads -inf
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                if (r < nr) {
                    const int32_t idx = b_lo + r * 32 + lane - c;
                    int32_t v = src[idx < 0 ? 0 : idx];
                    v = idx < 0 ? NEG_R : v;
                    key[r] = max_plus(v, g, key[r]);
                }
            }
        }
    }
}

// Fast path of one full tile whose every shift stays inside the -inf pad (no bounds checks):
// per option one address add, RPT conflict-free LDS and RPT VIADDMNMX.
template <int K, int RPT>
__device__ __forceinline__ void tile_keys_fast(const int32_t *__restrict__ src_lane, int32_t b_lo,
                                               const int32_t (&gp)[K], const int32_t (&cc)[K],
                                               int32_t (&key)[RPT])
{
    {
        const int32_t *__restrict__ s = src_lane + (b_lo - cc[0]);
#pragma unroll
        for (int r = 0; r < RPT; ++r) key[r] = s[r * 32] + gp[0];
    }
#pragma unroll
    for (int k = 1; k < K; ++k) {
        const int32_t *__restrict__ s = src_lane + (b_lo - cc[k]);
#pragma unroll
        for (int r = 0; r < RPT; ++r) key[r] = max_plus(s[r * 32], gp[k], key[r]);
    }
}

// Choice word of a tile: the tags (low CB bits of every key) of its RPT rows, gathered with
// byte permutes. Row j's field sits at bit choice_shift(j) = 8 (j & 3) + CB (j >> 2); the final
// NOT turns every tag (15 - k) into k (all 32 bits are fields).
template <int RPT, int CB>
__device__ __forceinline__ uint32_t pack_choices(const int32_t (&key)[RPT])
{
    constexpr uint32_t FM = ((1u << CB) - 1u) * 0x01010101u;
    uint32_t w = 0;
#pragma unroll
    for (int m = 0; m < RPT / 4; ++m) {
        const uint32_t lo = __byte_perm((uint32_t)key[4 * m], (uint32_t)key[4 * m + 1], 0x0040);
        const uint32_t hi = __byte_perm((uint32_t)key[4 * m + 2], (uint32_t)key[4 * m + 3], 0x0040);
        const uint32_t q = __byte_perm(lo, hi, 0x5410);
        w |= (q & FM) << (CB * m);
    }
    return ~w;
}

// One tile t of frame i: keys from `cur`, stripped values to `nxt`, choice word to the plane.
// OWN: the warp's first tile, whose own cells' previous values are held in registers `own`
// (a cost-0 option 0 then needs no shared-memory read); `own` is refreshed with the new values.
template <int K, int MODE, bool OWN>
__device__ __forceinline__ void dp_tile(const DpParams &P, int32_t t, int32_t i, int32_t nrows, int32_t ntiles,
                                        int32_t gtiles, const int32_t *__restrict__ cur, int32_t *__restrict__ nxt,
                                        uint32_t *__restrict__ sch, uint32_t *__restrict__ gch,
                                        const int32_t (&gp)[K], const int32_t (&cc)[K], int32_t cmax, bool inplace,
                                        int lane, int32_t (&own)[(K <= 4) ? 16 : 8])
{
    constexpr int CB = (K <= 4) ? 2 : 4;
    constexpr int RPT = 32 / CB;
    const int32_t b_lo = t * RPT * 32;
    const int32_t nr = min(RPT, nrows - t * RPT);
    int32_t key[RPT];
    const bool fast = (nr == RPT) && (cmax <= b_lo + P.pad_words);
    // rows are [-pad_words, row_words) around `cur` / `nxt`; planes hold ntiles tiles per frame
    TCHECK(b_lo + RPT * 32 <= P.row_words);
    TCHECK(!fast || b_lo - cmax >= -P.pad_words);
    TCHECK(MODE != DP_SOLVE_SMEM || (int64_t)(i * ntiles + t) * 32 + 32 <= (int64_t)P.chs_words);
    TCHECK(MODE == DP_SOLVE_SMEM || t < gtiles);
    if (fast) {
        const int32_t *__restrict__ src = cur + lane + b_lo;
        if (OWN && cc[0] == 0) {
#pragma unroll
            for (int r = 0; r < RPT; ++r) key[r] = own[r] + gp[0];
        } else {
#pragma unroll
            for (int r = 0; r < RPT; ++r) key[r] = src[r * 32 - cc[0]] + gp[0];
        }
#pragma unroll
        for (int k = 1; k < K; ++k) {
            const int32_t *__restrict__ s = src - cc[k];
#pragma unroll
            for (int r = 0; r < RPT; ++r) key[r] = max_plus(s[r * 32], gp[k], key[r]);
        }
    } else {
        tile_keys<K, RPT>(cur, b_lo, nr, P.pad_words, gp, cc, lane, key);
    }
    if (inplace) __syncwarp();                            // all reads of this tile done
    int32_t *__restrict__ dst = nxt + b_lo + lane;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int32_t v = key[r] & ~15;
        if (OWN) own[r] = v;
        if (fast || r < nr) dst[r * 32] = v;
    }
    const uint32_t word = pack_choices<RPT, CB>(key);
    if (MODE == DP_SOLVE_SMEM)
        sch[(i * ntiles + t) * 32 + lane] = word;
    else
        gch[((int64_t)i * gtiles + t) * 32 + lane] = word;
}

// ---- NEXT-5: u16 DP rows -------------------------------------------------------
// For a window whose values fit 16 bits the row holds v = S + V0 as u16 -- two cells per 32-bit
// word, so one conflict-free LDS.32 per option serves TWO cells (the 4-byte shared-load
// instruction rate, not bytes, bounds the int32 rows: DESIGN.md §6). Eligibility (decided per
// window on the device, dp_window): every gain >= 0, every frame has a cost-0 option (so every
// cell b >= 0 is feasible and the only -inf cells are the pad below 0, stored as 0), and
// sum_i max_k g_ik + V0 <= 65535 with V0 = max g + 1 (a candidate built on a pad cell, at most
// max g, then loses to every real one, at least V0). Exactly the int32 recurrence and tie-break:
// the key becomes (v << 16) | (15 - k), compared unsigned.
// Layout of one row buffer X (int32 words [X - PW, X + RW)): pad0 = [X - PW, X - PW/2) (zeros),
// copy0 = X - PW/2 (word q = cells 2q, 2q+1), pad1 = [X + RW/2 - PW/2, X + RW/2) (zeros),
// copy1 = X + RW/2 (word q = cells 2q - 1, 2q: the row shifted by one cell, so an ODD shift is an
// aligned word read of copy1 and an even one of copy0). Lane l of pair-row r of tile t owns pair
// p = t RPT 16 + r 32 + l (cells 2p, 2p + 1); a tile spans the same RPT 32 cells as the int32 tile.
template <int K, int MODE>
__device__ __forceinline__ void dp_tile_u16(const DpParams &P, int32_t t, int32_t i, int32_t ntiles, int32_t gtiles,
                                            const uint32_t *__restrict__ c0, const uint32_t *__restrict__ c1,
                                            uint32_t *__restrict__ n0, uint16_t *__restrict__ n1h,
                                            uint32_t *__restrict__ sch, uint32_t *__restrict__ gch,
                                            const uint32_t (&gp)[K], const int32_t (&cc)[K], int32_t cmax,
                                            bool inplace, int lane)
{
    constexpr int CB = (K <= 4) ? 2 : 4;
    constexpr int RPT = 32 / CB;
    constexpr int R2 = RPT / 2;                           // pair-rows per tile
    const int32_t cells = P.row_words;                    // u16 cells per copy
    const int32_t hp = P.pad_words >> 1;                  // pad words per copy
    const int32_t b_lo = t * RPT * 32;
    const int32_t p0 = t * RPT * 16 + lane;
    const bool fast = cmax <= b_lo + 2 * hp;              // every read inside the row or its pad
    TCHECK(2 * (p0 + (R2 - 1) * 32) + 1 < cells);
    TCHECK(MODE != DP_SOLVE_SMEM || (int64_t)(i * ntiles + t) * 32 + 32 <= (int64_t)P.chs_words);
    TCHECK(MODE == DP_SOLVE_SMEM || t < gtiles);
    uint32_t klo[R2], khi[R2];
    // option k of pair-row r: the word holding cells (2p - c, 2p + 1 - c) -> both candidate keys
    auto upd = [&](int k, int r, uint32_t wv) {
        const uint32_t lo = wv << 16, hi = wv & 0xffff0000u;
        if (k == 0) {
            klo[r] = lo + gp[0];
            khi[r] = hi + gp[0];
        } else {
            klo[r] = __viaddmax_u32(lo, gp[k], klo[r]);
            khi[r] = __viaddmax_u32(hi, gp[k], khi[r]);
        }
    };
    if (fast) {                                           // unchecked: every shift stays in the pad
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t *__restrict__ s = ((cc[k] & 1) ? c1 : c0) + (p0 - (cc[k] >> 1));
#pragma unroll
            for (int r = 0; r < R2; ++r) upd(k, r, s[r * 32]);
        }
    } else {                                              // low tiles: words below the pad read 0
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int32_t sh = cc[k] >> 1;
            const uint32_t *__restrict__ s = ((cc[k] & 1) ? c1 : c0) + (p0 - sh);
#pragma unroll
            for (int r = 0; r < R2; ++r) {
                const int32_t q = p0 + r * 32 - sh;
                upd(k, r, q >= -hp ? s[q < -hp ? 0 : r * 32] : 0u);
            }
        }
    }
    if (inplace) __syncwarp();                            // all reads of this tile done
    uint32_t *__restrict__ d0 = n0 + p0;
    uint16_t *__restrict__ d1 = n1h + 2 * p0 + 1;         // copy1 u16 index of cell 2p is 2p + 1
    int32_t key[RPT];
#pragma unroll
    for (int r = 0; r < R2; ++r) {
        d0[r * 32] = __byte_perm(klo[r], khi[r], 0x7632);
        d1[r * 64] = (uint16_t)(klo[r] >> 16);
        if (2 * (p0 + r * 32) + 2 < cells) d1[r * 64 + 1] = (uint16_t)(khi[r] >> 16);
        key[2 * r] = (int32_t)klo[r];
        key[2 * r + 1] = (int32_t)khi[r];
    }
    const uint32_t word = pack_choices<RPT, CB>(key);
    if (MODE == DP_SOLVE_SMEM)
        sch[(i * ntiles + t) * 32 + lane] = word;
    else
        gch[((int64_t)i * gtiles + t) * 32 + lane] = word;
}

// a5 of the long-window kernel (ONE window walked by one warp while the rest of the GPU idles:
// the round-trip latency is everything): one warp walks the HBM planes from (frame 0, b = C*) and
// resolves D frames per dependent round trip.
// Speculation: candidate q (lane q, or q - 32 in a lane's second slot) is a prefix
// (p_0 .. p_{d-1}) of d < D choices (q = 0: the empty prefix; then the K one-frame prefixes,
// the K^2 two-frame ones, ...). Costs do not depend on b,
// so each lane knows its cells b_j = b - sum_{l<j} c_{i+l, p_l} before the round, reads the
// choices at all of them at once, and decides ON ITS OWN whether its prefix is the realised one
// (every p_j equals the choice read at b_j). The realised deepest candidate holds the round:
// one ballot per slot and two shuffles hand its exits and its cost to the warp. Costs are loaded one
// round ahead, so the only dependent latency per round is one choice read + ballot + shuffle.
// (With many windows in flight -- the DP kernels and the standalone backtrack -- the walks share
// the load/store pipes and the extra loads cost more than the shorter chain saves: there
// backtrack_warp below is used.)
template <int K>
struct BtGeom {
    // candidates per lane (C) and frames per round (D): the largest D with sum_{j<D} K^j <= 32 C.
    // (C = 2, e.g. D = 3 for K = 6, measured slower on c4: the wider rounds cost more than the
    // saved round trips.)
    static constexpr int C = 1;
    static constexpr int D = (K == 2) ? 5 : (K <= 5 ? 3 : 2);
};

template <int K, int MODE, class CostF>
__device__ __forceinline__ void backtrack_warp_spec(int32_t N, int32_t b, const uint32_t *__restrict__ sch,
                                                    const uint32_t *__restrict__ gch, int32_t ntiles,
                                                    int32_t gtiles, CostF cost, uint8_t *__restrict__ exit_g,
                                                    uint8_t *__restrict__ exit_s, int lane)
{
    constexpr int CB = (K <= 4) ? 2 : 4;
    constexpr int RPT = 32 / CB;
    constexpr uint32_t CMASK = (1u << CB) - 1u;
    constexpr int D = BtGeom<K>::D;
    constexpr int C = BtGeom<K>::C;
    // decode each slot's candidate q = lane + 32 s: depth d (-1: idle) and digits (frame i first)
    int d[C];
    uint32_t dig[C];
#pragma unroll
    for (int sl = 0; sl < C; ++sl) {
        d[sl] = -1;
        dig[sl] = 0;
        int q = lane + 32 * sl, pw = 1;
#pragma unroll
        for (int dd = 0; dd < D; ++dd) {
            if (d[sl] < 0) {
                if (q < pw) {
                    d[sl] = dd;
                    int r = q;
                    for (int j = dd - 1; j >= 0; --j) {
                        dig[sl] |= (uint32_t)(r % K) << (4 * j);
                        r /= K;
                    }
                } else {
                    q -= pw;
                }
            }
            pw *= K;
        }
    }
    auto choice = [&](int32_t i, int32_t cell) -> int32_t {
        const int32_t t = cell / (32 * RPT);
        const int32_t j = (cell >> 5) & (RPT - 1);
        const uint32_t word = (MODE == DP_SOLVE_SMEM) ? sch[(i * ntiles + t) * 32 + (cell & 31)]
                                                      : gch[((int64_t)i * gtiles + t) * 32 + (cell & 31)];
        return (int32_t)((word >> choice_shift(j, CB)) & CMASK);
    };
    // costs of the round starting at frame i0, per slot: the prefix costs and every cost of frame
    // i0 + d
    auto load_costs = [&](int32_t i0, int32_t (&pcv)[C][D], int32_t (&lcv)[C][K]) {
#pragma unroll
        for (int sl = 0; sl < C; ++sl) {
#pragma unroll
            for (int j = 0; j < D - 1; ++j)
                pcv[sl][j] = (j < d[sl] && i0 + j < N) ? cost(i0 + j, (int)((dig[sl] >> (4 * j)) & 15u)) : 0;
            pcv[sl][D - 1] = 0;
            const bool last = d[sl] >= 0 && i0 + d[sl] < N;
#pragma unroll
            for (int k = 0; k < K; ++k) lcv[sl][k] = last ? cost(i0 + d[sl], k) : 0;
        }
    };
    // one round at frame i with this round's costs; prefetches the next round's into (pcn, lcn).
    // Returns false when the walk is over.
    auto round = [&](int32_t i, const int32_t (&pcv)[C][D], const int32_t (&lcv)[C][K], int32_t (&pcn)[C][D],
                     int32_t (&lcn)[C][K]) -> bool {
        const int32_t dm = min(D, N - i);
        if (i + D < N) load_costs(i + D, pcn, lcn);           // next round's costs, off the chain
        // the choices at every cell of each slot's prefix: D unconditional loads per slot
        // (clamped to a valid cell and frame) so they are all in flight at once
        int32_t kv[C][D], bd[C];
        bool neg[C];
#pragma unroll
        for (int sl = 0; sl < C; ++sl) {
            int32_t bj = b;
            bd[sl] = b;
            neg[sl] = false;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                kv[sl][j] = choice(min(i + j, N - 1), max(bj, 0));
                if (j <= d[sl]) neg[sl] |= bj < 0;
                if (j == d[sl]) bd[sl] = bj;
                if (j < D - 1 && j < d[sl]) bj -= pcv[sl][j];
            }
        }
        uint32_t packed_v[C];
        int32_t step_v[C];
        unsigned mask[C];
#pragma unroll
        for (int sl = 0; sl < C; ++sl) {
            bool on = d[sl] >= 0 && d[sl] == dm - 1 && !neg[sl];
            int32_t kd = 0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
                if (j < d[sl]) on = on && kv[sl][j] == (int32_t)((dig[sl] >> (4 * j)) & 15u);
                if (j == d[sl]) kd = kv[sl][j];
            }
            int32_t lk = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) lk = (k == kd) ? lcv[sl][k] : lk;
            mask[sl] = __ballot_sync(0xffffffffu, on);
            packed_v[sl] = dig[sl] | ((uint32_t)kd << (4 * (d[sl] < 0 ? 0 : d[sl])));
            step_v[sl] = (b - bd[sl]) + lk;
        }
        // the realised candidate: its slot (warp-uniform) and lane
        int ws = 0;
        unsigned m = mask[0];
#pragma unroll
        for (int sl = 1; sl < C; ++sl)
            if (m == 0) {
                ws = sl;
                m = mask[sl];
            }
        uint32_t pk = packed_v[0];
        int32_t st = step_v[0];
#pragma unroll
        for (int sl = 1; sl < C; ++sl)
            if (ws == sl) {
                pk = packed_v[sl];
                st = step_v[sl];
            }
        const int src = (__ffs(m) - 1) & 31;
        const uint32_t packed = __shfl_sync(0xffffffffu, pk, src);
        const int32_t step = __shfl_sync(0xffffffffu, st, src);
        if (m == 0) {                                         // unreachable for a consistent plane
            if (lane == 0)
                for (int32_t x = i; x < N; ++x) {
                    exit_g[x] = 0;
                    if (exit_s) exit_s[x] = 0;
                }
            return false;
        }
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < D; ++j)
                if (j < dm) {
                    const uint8_t k = (uint8_t)((packed >> (4 * j)) & 15u);
                    exit_g[i + j] = k;
                    if (exit_s) exit_s[i + j] = k;
                }
        }
        b -= step;
        return i + D < N;
    };
    // rounds alternate between two cost register sets (no copies of in-flight loads)
    int32_t pcA[C][D], lcA[C][K], pcB[C][D], lcB[C][K];
    load_costs(0, pcA, lcA);
    for (int32_t i = 0; i < N; i += 2 * D) {
        if (!round(i, pcA, lcA, pcB, lcB)) break;
        if (!round(i + D, pcB, lcB, pcA, lcA)) break;
    }
}

// a5 inside the DP kernel: warp 0 walks the choice planes from (frame 0, b = C*) and resolves
// D frames per dependent round trip. Costs do not depend on b, so while lane 0 reads frame i's
// choice at b, lane 1 + a reads frame i+1's at b - c_{i,a} and (D = 3, when 1 + K + K^2 <= 32)
// lane 1 + K + a K + a' reads frame i+2's at b - c_{i,a} - c_{i+1,a'}; shuffles then pick the
// realised branch. Lane 0 writes the exits (global, and shared when exit_s != nullptr).
// U16: planes written by dp_tile_u16 (a lane's tile word holds the choices of its cell PAIRS).
template <int K, int MODE, class CostF, bool U16 = false>
__device__ __forceinline__ void backtrack_warp(int32_t N, int32_t b, const uint32_t *__restrict__ sch,
                                               const uint32_t *__restrict__ gch, int32_t ntiles, int32_t gtiles,
                                               CostF cost, uint8_t *__restrict__ exit_g, uint8_t *__restrict__ exit_s,
                                               int lane)
{
    constexpr int CB = (K <= 4) ? 2 : 4;
    constexpr int RPT = 32 / CB;
    constexpr uint32_t CMASK = (1u << CB) - 1u;
    constexpr int D = (1 + K + K * K <= 32) ? 3 : 2;
    int depth = -1, a = 0, a2 = 0;
    if (lane == 0) {
        depth = 0;
    } else if (lane <= K) {
        depth = 1;
        a = lane - 1;
    } else if (D == 3 && lane <= K + K * K) {
        depth = 2;
        a = (lane - 1 - K) / K;
        a2 = (lane - 1 - K) % K;
    }
    auto choice = [&](int32_t i, int32_t cell) -> int32_t {
        const int32_t t = cell / (32 * RPT);
        int32_t ln, j;
        if (U16) {                                    // cell q of the tile: pair q/2 = (row, lane)
            const int32_t q = cell - t * 32 * RPT;
            ln = (q >> 1) & 31;
            j = 2 * (q >> 6) + (q & 1);
        } else {
            ln = cell & 31;
            j = (cell >> 5) & (RPT - 1);
        }
        TCHECK(cell >= 0 && i >= 0 && i < N && t < (MODE == DP_SOLVE_SMEM ? ntiles : gtiles));
        const uint32_t word = (MODE == DP_SOLVE_SMEM) ? sch[(i * ntiles + t) * 32 + ln]
                                                      : gch[((int64_t)i * gtiles + t) * 32 + ln];
        return (int32_t)((word >> choice_shift(j, CB)) & CMASK);
    };
    auto emit = [&](int32_t i, int32_t k) {
        exit_g[i] = (uint8_t)k;
        if (exit_s) exit_s[i] = (uint8_t)k;
    };
    int32_t i = 0;
    // full rounds: the deepest lane whose speculated prefix matches the realised choices holds
    // the whole round -- one vote and two shuffles resolve it (no serial shuffle chain)
    for (; i + D <= N; i += D) {
        const int32_t ca = depth >= 1 ? cost(i, a) : 0;
        const int32_t cb = depth == 2 ? cost(i + 1, a2) : 0;
        int32_t kk = 0;
        if (depth >= 0) {
            const int32_t bt = b - ca - cb;
            kk = bt >= 0 ? choice(i + depth, bt) : 0;
        }
        const int32_t k0 = __shfl_sync(0xffffffffu, kk, 0);
        const int32_t k1 = __shfl_sync(0xffffffffu, kk, D == 3 && depth == 2 ? 1 + a : lane);
        const bool on_path = (depth == D - 1) && (a == k0) && (D == 2 || a2 == k1);
        int32_t packed = 0, step = 0;
        if (on_path) {
            step = ca + cb + cost(i + depth, kk);
            packed = D == 3 ? (k0 | (k1 << 4) | (kk << 8)) : (k0 | (kk << 4));
        }
        const int src = __ffs(__ballot_sync(0xffffffffu, on_path)) - 1;
        packed = __shfl_sync(0xffffffffu, packed, src);
        step = __shfl_sync(0xffffffffu, step, src);
        if (lane == 0) {
            emit(i, packed & 15);
            emit(i + 1, (packed >> 4) & 15);
            if (D == 3) emit(i + 2, (packed >> 8) & 15);
        }
        b -= step;
    }
    // tail (< D frames): plain walk by lane 0
    if (lane == 0) {
        for (; i < N; ++i) {
            const int32_t k = choice(i, b);
            emit(i, k);
            b -= cost(i, k);
        }
    }
}

// a5 for any K (runtime value): the warp walk of backtrack_warp with the same speculation -- lane 0
// reads frame i at b, lanes 1..K frame i+1 at b - c_{i,a}, and (when 1 + K + K^2 <= 32, i.e.
// K <= 5) lanes 1+K+aK+a' frame i+2 at b - c_{i,a} - c_{i+1,a'} -- compiled once for all K, so a
// kernel walking windows of many K values keeps one small body in the instruction cache.
template <class CostF>
__device__ __forceinline__ void backtrack_warp_rt(const int K, int32_t N, int32_t b, const uint32_t *__restrict__ gch,
                                                  int32_t gtiles, CostF cost, uint8_t *__restrict__ exit_g, int lane)
{
    const int CB = K <= 4 ? 2 : 4;
    const int lg_tile = K <= 4 ? 9 : 8;                  // log2(32 * RPT)
    const int rmask = K <= 4 ? 15 : 7;                   // RPT - 1
    const uint32_t cmask = (1u << CB) - 1u;
    const int D = (1 + K + K * K <= 32) ? 3 : 2;
    int depth = -1, a = 0, a2 = 0;
    if (lane == 0) {
        depth = 0;
    } else if (lane <= K) {
        depth = 1;
        a = lane - 1;
    } else if (D == 3 && lane <= K + K * K) {
        depth = 2;
        a = (lane - 1 - K) / K;
        a2 = (lane - 1 - K) % K;
    }
    auto choice = [&](int32_t i, int32_t cell) -> int32_t {
        TCHECK(cell >= 0 && i >= 0 && i < N && (cell >> lg_tile) < gtiles);
        const uint32_t word = gch[((int64_t)i * gtiles + (cell >> lg_tile)) * 32 + (cell & 31)];
        return (int32_t)((word >> choice_shift((cell >> 5) & rmask, CB)) & cmask);
    };
    int32_t i = 0;
    for (; i + D <= N; i += D) {
        const int32_t ca = depth >= 1 ? cost(i, a) : 0;
        const int32_t cb = depth == 2 ? cost(i + 1, a2) : 0;
        int32_t kk = 0;
        if (depth >= 0) {
            const int32_t bt = b - ca - cb;
            kk = bt >= 0 ? choice(i + depth, bt) : 0;
        }
        const int32_t k0 = __shfl_sync(0xffffffffu, kk, 0);
        const int32_t k1 = __shfl_sync(0xffffffffu, kk, D == 3 && depth == 2 ? 1 + a : lane);
        const bool on_path = (depth == D - 1) && (a == k0) && (D == 2 || a2 == k1);
        int32_t packed = 0, step = 0;
        if (on_path) {
            step = ca + cb + cost(i + depth, kk);
            packed = D == 3 ? (k0 | (k1 << 4) | (kk << 8)) : (k0 | (kk << 4));
        }
        const int src = __ffs(__ballot_sync(0xffffffffu, on_path)) - 1;
        packed = __shfl_sync(0xffffffffu, packed, src);
        step = __shfl_sync(0xffffffffu, step, src);
        if (lane == 0) {
            exit_g[i] = (uint8_t)(packed & 15);
            exit_g[i + 1] = (uint8_t)((packed >> 4) & 15);
            if (D == 3) exit_g[i + 2] = (uint8_t)((packed >> 8) & 15);
        }
        b -= step;
    }
    if (lane == 0) {
        for (; i < N; ++i) {
            const int32_t k = choice(i, b);
            exit_g[i] = (uint8_t)k;
            b -= cost(i, k);
        }
    }
}

// a6 fused: accumulate one window's plan statistics (turbo.h layout) into the per-GPU vector.
// The CTA-private histogram `hist` (176 u32) was filled by thread 0; every counter goes to
// global memory with one fire-and-forget reduction (RED) per non-zero entry.
__device__ __forceinline__ void flush_window_stats(const DpParams &P, uint32_t *__restrict__ hist, int32_t G,
                                                   int32_t Cst, bool feas, int32_t N, int tid, int nthr)
{
    unsigned long long *st = reinterpret_cast<unsigned long long *>(P.stats);
    for (int x = tid; x < 176; x += nthr) {
        const uint32_t v = hist[x];
        if (v) atomicAdd(&st[x], (unsigned long long)v);
    }
    if (tid == 0) {
        atomicAdd(&st[176], (unsigned long long)(long long)G);
        atomicAdd(&st[177], (unsigned long long)(long long)Cst);
        atomicAdd(&st[178], 1ull);
        atomicAdd(&st[179], (unsigned long long)N);
        if (!feas) atomicAdd(&st[180], 1ull);
    }
}

// OSM: the window's options staged in shared memory as packed (g << 4 | 15 - k, c) pairs and read
// with broadcast LDS.64; otherwise lane q*K + k holds option k of a chunk of frames (prefetched a
// chunk ahead) and the warp broadcasts it with shuffles (windows whose option table does not fit).
// FUSE (turbo_schedule): a1 (budget from capacity) and a2 (options straight from class ids and
// the profile, never materialised in HBM) in the prologue, a6 (statistics) in the epilogue.
// U16: windows that qualify (decided on the device, see dp_tile_u16) run the u16-row body.
template <int K, int MODE, bool OSM, bool FUSE, bool U16 = false>
__device__ __forceinline__ void dp_window(const DpParams &P, int64_t w, int32_t *__restrict__ rowA,
                                          int32_t *__restrict__ rowB, uint32_t *__restrict__ sch,
                                          int32_t *__restrict__ cst, int2 *__restrict__ opt_s,
                                          int64_t *__restrict__ red, uint32_t *__restrict__ hist, int warp,
                                          int nwarps, int lane)
{
    constexpr int CB = (K <= 4) ? 2 : 4;          // choice bits
    constexpr int RPT = 32 / CB;                   // rows of 32 cells per tile (per choice word)
    static_assert(!U16 || (OSM && MODE != DP_PLAN), "u16 rows: staged options, walk in the kernel");
    const bool inplace = (nwarps == 1);
    const int tid = warp * 32 + lane;
    const int nthr = nwarps * 32;

    trace_mark(P, w, 0);
    const turbo_window_t *win = P.windows + w;
    const int64_t ff = win->first_frame;
    const int64_t fo = win->first_option;
    const int32_t N = win->num_frames;
    int32_t B = win->budget;
    const int32_t Bb = win->budget_bound;
    const int64_t choff = win->choice_offset;

    const int32_t *__restrict__ og = P.opt_gain + fo;
    const int32_t *__restrict__ oc = P.opt_cost + fo;
    // option (g, c) of frame i, exit k straight from global memory: the option table (lookup
    // path) or, fused, the profile row of the frame's class (a zero row for a class >= C)
    int32_t prof_C = 0;
    const int32_t *prof_g = nullptr, *prof_c = nullptr;
    if (FUSE) {
        const turbo_profile_t *prof = P.profiles + win->profile;
        prof_C = prof->num_classes;
        prof_g = prof->gain;
        prof_c = prof->cost;
    }
    auto load_opt = [&](int32_t i, int32_t k, int32_t &g, int32_t &c) {
        if (FUSE) {
            const int32_t cls = frame_class(P, ff + i, prof_C);
            if (cls < prof_C) {
                g = __ldg(prof_g + cls * K + k);
                c = __ldg(prof_c + cls * K + k);
            } else {
                g = 0;
                c = 0;
            }
        } else {
            g = __ldg(og + (int64_t)i * K + k);
            c = __ldg(oc + (int64_t)i * K + k);
        }
    };
    auto class_of = [&](int32_t i) -> uint32_t {               // fused statistics only
        return OSM ? reinterpret_cast<const uint8_t *>(opt_s + P.max_options + P.prof_entries)[i]
                   : (uint32_t)frame_class(P, ff + i, prof_C);
    };

    if (FUSE) {
        // a1 (reading R3): B_w = max(0, capacity_w - m_w * u0)
        if (P.capacity != nullptr) {
            const int64_t b = (int64_t)P.capacity[w] - (int64_t)N * (int64_t)P.base_cost;
            B = (int32_t)(b < 0 ? 0 : (b > 0x7fffffffll ? 0x7fffffff : b));
            if (tid == 0) P.windows_rw[w].budget = B;
        }
        for (int x = tid; x < 176; x += nthr) hist[x] = 0;
        if (P.theta != nullptr)                           // NEXT-3 fused: the classes, for the walk / stats
            for (int32_t x = tid; x < N; x += nthr) P.class_out[ff + x] = (uint8_t)frame_class(P, ff + x, prof_C);
    }

    // ---- prologue: stage options (OSM), validate, sums for the infeasible report (reading R8)
    bool bad = (B < 0) || (B > Bb);
    if (OSM) {
        const int32_t n_opt = N * K;
        if (FUSE) {
            // a2: the option row of frame i is the profile row of its
            // class. Class ids and the profile table are loaded concurrently into shared memory
            // (one global latency), then every option is a shared-memory gather.
            const turbo_profile_t &pr = P.profiles[win->profile];
            const int32_t C = pr.num_classes;
            const int32_t *__restrict__ pg = pr.gain;
            const int32_t *__restrict__ pc = pr.cost;
            int2 *__restrict__ prof_s = opt_s + P.max_options;
            uint8_t *__restrict__ cls_s = reinterpret_cast<uint8_t *>(prof_s + P.prof_entries);
            for (int32_t x = tid; x < N; x += nthr) cls_s[x] = (uint8_t)frame_class(P, ff + x, C);
            for (int32_t x = tid; x < C * K; x += nthr) prof_s[x] = make_int2(__ldg(pg + x), __ldg(pc + x));
            if (nwarps > 1) __syncthreads(); else __syncwarp();
            for (int32_t o = tid; o < n_opt; o += nthr) {
                const int32_t i = o / K;
                const int32_t k = o - i * K;
                const int32_t cls = cls_s[i];
                int32_t g = 0, c = 0;
                if (cls < C) {
                    const int2 v = prof_s[cls * K + k];
                    g = v.x;
                    c = v.y;
                } else if (k == 0) {
                    atomic_min_i64(&P.status[0], ff + i);
                }
                bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
                opt_s[o] = make_int2((g << 4) | (15 - k), c);
            }
        } else {
            for (int32_t o = tid; o < n_opt; o += nthr) {
                const int32_t g = __ldg(og + o);
                const int32_t c = __ldg(oc + o);
                bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
                const int32_t k = o % K;
                opt_s[o] = make_int2((g << 4) | (15 - k), c);
            }
        }
        if (nwarps > 1)
            bad = __syncthreads_or(bad);
        else
            bad = __any_sync(0xffffffffu, bad);
    }
    if (warp == 0) {
        int64_t abs_sum = 0, g0_sum = 0, c0_sum = 0;
        bool u_ok = true;                                 // U16: gains >= 0, a cost-0 option per frame
        int32_t u_gmax = 0;
        for (int32_t i = lane; i < N; i += 32) {
            int32_t m = 0;
            bool zc = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                int32_t g, c;
                if (OSM) {
                    const int2 v = opt_s[i * K + k];
                    g = v.x >> 4;
                    c = v.y;
                } else {
                    load_opt(i, k, g, c);
                    bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
                    if (FUSE && k == 0 && frame_class(P, ff + i, prof_C) >= prof_C)
                        atomic_min_i64(&P.status[0], ff + i);
                }
                const int32_t a = g < 0 ? -g : g;
                m = a > m ? a : m;
                if (k == 0) {
                    g0_sum += g;
                    c0_sum += c;
                }
                if (U16) {
                    u_ok = u_ok && g >= 0;
                    zc = zc || c == 0;
                    u_gmax = max(u_gmax, g);
                }
            }
            abs_sum += m;
            u_ok = u_ok && zc;
        }
        abs_sum = warp_sum_i64(abs_sum);
        g0_sum = warp_sum_i64(g0_sum);
        c0_sum = warp_sum_i64(c0_sum);
        bad = __any_sync(0xffffffffu, bad) || abs_sum >= GAIN_RANGE_LIMIT || c0_sum >= 0x7fffffffll;
        if (U16) {
            u_ok = __all_sync(0xffffffffu, u_ok);
            u_gmax = (int32_t)__reduce_max_sync(0xffffffffu, (uint32_t)u_gmax);
        }
        if (lane == 0) {
            red[0] = bad ? 1 : 0;
            red[1] = g0_sum;
            red[2] = c0_sum;
            red[3] = 0;                                   // C* counter
            // U16: V0 = max g + 1 when sum_i max_k g_ik + V0 fits 16 bits, else 0 (int32 rows)
            red[4] = (U16 && P.u16 && N > 0 && u_ok && abs_sum + u_gmax + 1 <= 65535) ? u_gmax + 1 : 0;
        }
    }
    const int32_t ntiles = (((B + 32) >> 5) + RPT - 1) / RPT;
    // rows are computed in whole tiles: the cells above B (up to the tile edge, inside the row
    // allocation) are garbage nobody valid reads (cell b only reads cells <= b), and every tile
    // takes the unpredicated path
    const int32_t nrows = ntiles * RPT;
    // S_N = 0 on every cell (including the padding cells above B)
    for (int32_t x = tid; x < nrows * 32; x += nthr) rowA[x] = 0;
    if (nwarps > 1) __syncthreads(); else __syncwarp();
    if (red[0]) {
        if (tid == 0) {
            P.best_gain[w] = 0;
            P.best_cost[w] = 0;
            P.feasible[w] = 0;
            atomic_min_i64(&P.status[1], w);
        }
        if (MODE != DP_PLAN)
            for (int32_t i = tid; i < N; i += nthr) P.exit_out[ff + i] = 0;
        if (FUSE && MODE != DP_PLAN) {                    // (plan mode: the walk kernel counts it)
            if (tid == 0)
                for (int32_t i = 0; i < N; ++i) {
                    const uint32_t cls = class_of(i);
                    hist[0] += 1;
                    if (cls < 10) hist[16 + cls * 16] += 1;
                }
            if (nwarps > 1) __syncthreads(); else __syncwarp();
            flush_window_stats(P, hist, 0, 0, false, N, tid, nthr);
        }
        return;
    }

    trace_mark(P, w, 1);
    if (P.debug & 64) return;                         // timing: prologue only
    // choice-plane stride (tiles per frame): the layout bound for HBM planes, exact for smem
    const int32_t gtiles = (int32_t)(((Bb + 32) >> 5) + RPT - 1) / RPT;
    uint32_t *__restrict__ gch = reinterpret_cast<uint32_t *>(P.workspace + choff);

    // ---- a5 fused: forward backtrack from (frame 0, b = C*); a6 (fused): statistics
    // (shared by the int32 and the u16 bodies; u16 planes use the pair mapping)
    auto finish = [&](int32_t G, int32_t Cst, bool feas, bool u16) {
        uint8_t *exit_s = nullptr;                        // fused + staged options: exits in smem
        if (FUSE && OSM)
            exit_s = reinterpret_cast<uint8_t *>(opt_s + P.max_options + P.prof_entries) + ((N + 3) & ~3);
        if (!feas) {
            for (int32_t i = tid; i < N; i += nthr) {
                P.exit_out[ff + i] = 0;
                if (exit_s) exit_s[i] = 0;
            }
        } else if (warp == 0 && !(P.debug & 16)) {
            // costs of the walk: the staged table, or global memory (option table / profile row)
            auto cost = [&](int32_t i, int32_t k) -> int32_t {
                if (OSM) return opt_s[i * K + k].y;
                int32_t g, c;
                load_opt(i, k, g, c);
                return c;
            };
            bool done = false;
            if constexpr (U16) {
                if (u16) {
                    backtrack_warp<K, MODE, decltype(cost), true>(N, Cst, sch, gch, ntiles, gtiles, cost,
                                                                  P.exit_out + ff, exit_s, lane);
                    done = true;
                }
            }
            if (done) {
            } else if (MODE == DP_SOLVE_SMEM && OSM && (P.debug & 256)) {
                backtrack_warp_spec<K, MODE>(N, Cst, sch, gch, ntiles, gtiles, cost, P.exit_out + ff, exit_s, lane);
            } else {
                backtrack_warp<K, MODE>(N, Cst, sch, gch, ntiles, gtiles, cost, P.exit_out + ff, exit_s, lane);
            }
        }
        if (FUSE) {                                       // a6: CTA-private histograms
            if (nwarps > 1) __syncthreads(); else __syncwarp();
            trace_mark(P, w, 4);
            for (int32_t i = tid; i < N; i += nthr) {
                const uint32_t k = exit_s ? exit_s[i] : P.exit_out[ff + i];   // global: visible after the barrier
                const uint32_t cls = class_of(i);
                atomicAdd(&hist[k], 1u);
                if (cls < 10) atomicAdd(&hist[16 + cls * 16 + k], 1u);
            }
            if (nwarps > 1) __syncthreads(); else __syncwarp();
            if (!(P.debug & 8)) flush_window_stats(P, hist, G, Cst, feas, N, tid, nthr);
        }
    };

    if constexpr (U16) {
        if (red[4] != 0) {
            // ---- NEXT-5: the u16-row body (dp_tile_u16). Options restaged as (g << 16 | 15 - k, c).
            const uint32_t V0 = (uint32_t)red[4];
            if (tid == 0 && P.u16_count != nullptr)
                atomicAdd(reinterpret_cast<unsigned long long *>(P.u16_count), 1ull);
            for (int32_t o = tid; o < N * K; o += nthr) {
                const int32_t x = opt_s[o].x;
                opt_s[o].x = (int32_t)(((uint32_t)(x >> 4) << 16) | (uint32_t)(x & 15));
            }
            const int32_t PW = P.pad_words, RW = P.row_words, HP = PW >> 1, HR = RW >> 1;
            uint32_t *const A0 = reinterpret_cast<uint32_t *>(rowA) - HP;
            uint32_t *const A1 = reinterpret_cast<uint32_t *>(rowA) + HR;
            uint32_t *const B0 = reinterpret_cast<uint32_t *>(rowB) - HP;
            uint32_t *const B1 = reinterpret_cast<uint32_t *>(rowB) + HR;
            for (int32_t x = tid; x < HP; x += nthr) {    // pads: 0 = -inf (below every real v >= V0)
                A0[x - HP] = 0;
                A1[x - HP] = 0;
                if (nwarps > 1) {
                    B0[x - HP] = 0;
                    B1[x - HP] = 0;
                }
            }
            const uint32_t VV = V0 | (V0 << 16);          // S_N = 0 -> v = V0 on every cell b >= 0
            for (int32_t x = tid; x < nrows * 16; x += nthr) {
                A0[x] = VV;
                A1[x] = x == 0 ? (V0 << 16) : VV;         // copy1 word 0 = (cell -1 = pad, cell 0)
            }
            if (nwarps > 1 && tid == 0) B1[0] = 0;        // cell -1 of the other buffer's copy1
            if (nwarps > 1) __syncthreads(); else __syncwarp();
            const uint32_t *c0 = A0, *c1 = A1;
            uint32_t *n0 = inplace ? A0 : B0, *n1 = inplace ? A1 : B1;
            const int32_t t0 = inplace ? ntiles - 1 : warp;
            const int32_t dt = inplace ? -1 : nwarps;
            for (int32_t i = N - 1; i >= 0; --i) {
                uint32_t gp[K];
                int32_t cc[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int2 v = opt_s[i * K + k];
                    gp[k] = (uint32_t)v.x;
                    cc[k] = v.y;
                }
                int32_t cmax = cc[0];
#pragma unroll
                for (int k = 1; k < K; ++k) cmax = max(cmax, cc[k]);
                for (int32_t t = t0; t >= 0 && t < ntiles; t += dt)
                    dp_tile_u16<K, MODE>(P, t, i, ntiles, gtiles, c0, c1, n0, reinterpret_cast<uint16_t *>(n1), sch,
                                         gch, gp, cc, cmax, inplace, lane);
                if (nwarps > 1) __syncthreads(); else __syncwarp();
                const uint32_t *t_0 = c0, *t_1 = c1;
                c0 = n0;
                c1 = n1;
                n0 = const_cast<uint32_t *>(t_0);
                n1 = const_cast<uint32_t *>(t_1);
            }
            trace_mark(P, w, 2);
            // a4 on v = S_0 + V0 (every cell >= 0 feasible under the eligibility rule)
            const uint16_t *v = reinterpret_cast<const uint16_t *>(c0);
            const int32_t vB = v[B];
            const bool feas = vB >= (int32_t)V0;
            const int32_t cnt = (warp == 0 && feas) ? warp_first_at_least(v, B, vB, lane) : 0;
            const int32_t G = feas ? vB - (int32_t)V0 : (int32_t)red[1];
            const int32_t Cst = feas ? cnt : (int32_t)red[2];
            if (tid == 0) {
                P.best_gain[w] = G;
                P.best_cost[w] = Cst;
                P.feasible[w] = feas ? 1 : 0;
            }
            trace_mark(P, w, 3);
            finish(G, Cst, feas, true);
            // the int32 rows' -inf pads back for the CTA's next window
            if (nwarps > 1) __syncthreads(); else __syncwarp();
            for (int32_t x = tid; x < PW; x += nthr) {
                rowA[x - PW] = NEG_R;
                if (nwarps > 1) rowB[x - PW] = NEG_R;
            }
            return;
        }
    }

    // !OSM: options live in registers, CH = 32/K frames per warp-wide chunk (lane q*K + k holds
    // option k of the chunk's q-th frame); the next chunk is loaded while the current one is
    // consumed, so CH frames of work hide the global-load latency.
    constexpr int CH = 32 / K;
    // Pipeline (no load is consumed before a whole chunk of frames has been computed):
    // a = current chunk (packed keys), b = next chunk (raw values, as loaded), n_cls = class ids of
    // the chunk after next (fused: the profile row address of chunk m+1 needs chunk m+1's class).
    int32_t a_gp = 0, a_c = 0, b_g = 0, b_c = 0, n_cls = 0;
    bool b_ok = true;
    const int lq = lane / K, lk = lane - (lane / K) * K;
    auto load_cls = [&](int32_t hi) -> int32_t {               // frames hi, hi-1, ... of a chunk
        const int32_t i = hi - lq;
        return (FUSE && lq < CH && i >= 0) ? frame_class(P, ff + i, prof_C) : 0;
    };
    auto load_raw = [&](int32_t hi, int32_t cls, int32_t &g, int32_t &c, bool &ok) {
        const int32_t i = hi - lq;
        g = 0;
        c = 0;
        ok = true;
        if (lq < CH && i >= 0) {
            if (FUSE) {                                        // a class >= C reads as a zero row
                ok = cls < prof_C;
                const int32_t row = ok ? cls : 0;
                g = __ldg(prof_g + row * K + lk);
                c = __ldg(prof_c + row * K + lk);
            } else {
                g = __ldg(og + (int64_t)i * K + lk);
                c = __ldg(oc + (int64_t)i * K + lk);
            }
        }
    };
    auto pack = [&](int32_t g, int32_t c, bool ok) {
        a_gp = ((ok ? g : 0) << 4) | (15 - lk);
        a_c = ok ? c : 0;
    };
    if (!OSM && N > 0) {
        int32_t g, c;
        bool ok;
        load_raw(N - 1, load_cls(N - 1), g, c, ok);                 // chunk 0 (the one wait)
        pack(g, c, ok);
        load_raw(N - 1 - CH, load_cls(N - 1 - CH), b_g, b_c, b_ok);  // chunk 1
        n_cls = load_cls(N - 1 - 2 * CH);                            // chunk 2's classes
    }
    int32_t *__restrict__ cur = rowA;
    int32_t *__restrict__ nxt = inplace ? rowA : rowB;
    int32_t own[RPT];                                      // S_{i+1} of the warp's first tile
#pragma unroll
    for (int r = 0; r < RPT; ++r) own[r] = 0;
    // in place: top-down so a tile's reads never see the updated tiles above it
    const int32_t t0 = inplace ? ntiles - 1 : warp;
    const int32_t dt = inplace ? -1 : nwarps;

    for (int32_t i = N - 1; i >= 0; --i) {
        int32_t gp[K], cc[K];
        TCHECK(!OSM || (i + 1) * K <= P.max_options);
        if (OSM) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int2 v = opt_s[i * K + k];
                gp[k] = v.x;
                cc[k] = v.y;
            }
        } else {
            const int32_t f = N - 1 - i;
            const int q = f % CH;
            if (q == 0 && f > 0) {                        // next chunk becomes current; prefetch
                pack(b_g, b_c, b_ok);
                load_raw(i - CH, n_cls, b_g, b_c, b_ok);
                n_cls = load_cls(i - 2 * CH);
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                gp[k] = __shfl_sync(0xffffffffu, a_gp, q * K + k);
                cc[k] = __shfl_sync(0xffffffffu, a_c, q * K + k);
            }
        }
        int32_t cmax = cc[0];
#pragma unroll
        for (int k = 1; k < K; ++k) cmax = max(cmax, cc[k]);
        if (t0 < ntiles)
            dp_tile<K, MODE, true>(P, t0, i, nrows, ntiles, gtiles, cur, nxt, sch, gch, gp, cc, cmax, inplace, lane,
                                   own);
        for (int32_t t = t0 + dt; t >= 0 && t < ntiles; t += dt)
            dp_tile<K, MODE, false>(P, t, i, nrows, ntiles, gtiles, cur, nxt, sch, gch, gp, cc, cmax, inplace, lane,
                                    own);
        if (nwarps > 1) __syncthreads(); else __syncwarp();   // frame i visible to frame i-1
        int32_t *tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    // after the swap `cur` holds S_0 (in place: cur == nxt == rowA)
    trace_mark(P, w, 2);

    // ---- a4: optimum extraction (C* by warp 0, the warp that walks; nobody else needs it)
    const int32_t RB = cur[B];
    const bool feas = RB > VALID_MIN_R;
    const int32_t cnt = (warp == 0 && feas) ? warp_first_at_least(cur, B, RB, lane) : 0;
    const int32_t G = feas ? (RB >> 4) : (int32_t)red[1];
    const int32_t Cst = feas ? cnt : (int32_t)red[2];
    if (tid == 0) {
        P.best_gain[w] = G;
        P.best_cost[w] = Cst;
        P.feasible[w] = feas ? 1 : 0;
    }
    trace_mark(P, w, 3);
    if (MODE == DP_PLAN) return;
    finish(G, Cst, feas, false);
}

// Out-of-line instance per K for the mixed-K kernel: keeps that kernel a small switch over
// separately compiled bodies (compile time, register allocation per K).
template <int K, int MODE, bool OSM, bool FUSE>
__device__ __noinline__ void dp_window_call(const DpParams &P, int64_t w, int32_t *rowA, int32_t *rowB,
                                            uint32_t *sch, int32_t *cst, int2 *opt_s, int64_t *red, uint32_t *hist,
                                            int warp, int nwarps, int lane)
{
    dp_window<K, MODE, OSM, FUSE>(P, w, rowA, rowB, sch, cst, opt_s, red, hist, warp, nwarps, lane);
}

// Generic-K body of the mixed-K kernel in plan mode (choice planes to HBM; the walk runs in its own
// kernel). K is a runtime value: ONE body per choice width (CB = 2 for K <= 4, 4 otherwise) instead
// of fifteen unrolled ones. Measured on c5: with windows of 15 different K sharing an SM, the
// per-K bodies thrash the instruction cache (ncu: 37 "no instruction" stalls per issued
// instruction in the short-row launch) -- these windows are latency-bound, so the option loop
// that is not unrolled costs nothing there. Same recurrence, packed keys and outputs as dp_window.
template <int CB, bool OSM, bool FUSE>
__device__ __forceinline__ void dp_window_gen(const DpParams &P, int64_t w, const int K, int32_t *__restrict__ rowA,
                                           int32_t *__restrict__ rowB, int2 *__restrict__ opt_s,
                                           int64_t *__restrict__ red, int warp, int nwarps, int lane)
{
    constexpr int RPT = 32 / CB;
    const bool inplace = (nwarps == 1);
    const int tid = warp * 32 + lane;
    const int nthr = nwarps * 32;
    const turbo_window_t *win = P.windows + w;
    const int64_t ff = win->first_frame;
    const int64_t fo = win->first_option;
    const int32_t N = win->num_frames;
    int32_t B = win->budget;
    const int32_t Bb = win->budget_bound;
    const int32_t *__restrict__ og = P.opt_gain + fo;
    const int32_t *__restrict__ oc = P.opt_cost + fo;
    int32_t prof_C = 0;
    const int32_t *prof_g = nullptr, *prof_c = nullptr;
    if (FUSE) {
        const turbo_profile_t *prof = P.profiles + win->profile;
        prof_C = prof->num_classes;
        prof_g = prof->gain;
        prof_c = prof->cost;
        if (P.capacity != nullptr) {     // a1 (reading R3): B_w = max(0, capacity_w - m_w u0)
            const int64_t b = (int64_t)P.capacity[w] - (int64_t)N * (int64_t)P.base_cost;
            B = (int32_t)(b < 0 ? 0 : (b > 0x7fffffffll ? 0x7fffffff : b));
            if (tid == 0) P.windows_rw[w].budget = B;
        }
        if (P.theta != nullptr)          // NEXT-3 fused: the classes, for the walk / stats kernels
            for (int32_t x = tid; x < N; x += nthr) P.class_out[ff + x] = (uint8_t)frame_class(P, ff + x, prof_C);
    }
    auto load_opt = [&](int32_t i, int32_t k, int32_t &g, int32_t &c) {
        if (FUSE) {                      // a2: the profile row of the frame's class (zero row for >= C)
            const int32_t cls = frame_class(P, ff + i, prof_C);
            g = cls < prof_C ? __ldg(prof_g + cls * K + k) : 0;
            c = cls < prof_C ? __ldg(prof_c + cls * K + k) : 0;
        } else {
            g = __ldg(og + (int64_t)i * K + k);
            c = __ldg(oc + (int64_t)i * K + k);
        }
    };
    // ---- prologue: stage options (OSM), validate, sums for the infeasible report (reading R8)
    bool bad = (B < 0) || (B > Bb);
    if (OSM) {
        for (int32_t o = tid; o < N * K; o += nthr) {
            const int32_t i = o / K, k = o - (o / K) * K;
            int32_t g, c;
            load_opt(i, k, g, c);
            bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
            opt_s[o] = make_int2((g << 4) | (15 - k), c);
        }
        bad = nwarps > 1 ? __syncthreads_or(bad) : __any_sync(0xffffffffu, bad);
    }
    if (warp == 0) {
        int64_t abs_sum = 0, g0_sum = 0, c0_sum = 0;
        for (int32_t i = lane; i < N; i += 32) {
            int32_t m = 0;
            if (FUSE && frame_class(P, ff + i, prof_C) >= prof_C) atomic_min_i64(&P.status[0], ff + i);
            for (int k = 0; k < K; ++k) {
                int32_t g, c;
                if (OSM) {
                    const int2 v = opt_s[i * K + k];
                    g = v.x >> 4;
                    c = v.y;
                } else {
                    load_opt(i, k, g, c);
                    bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
                }
                m = max(m, g < 0 ? -g : g);
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
        if (lane == 0) {
            red[0] = bad ? 1 : 0;
            red[1] = g0_sum;
            red[2] = c0_sum;
            red[3] = 0;
        }
    }
    const int32_t ntiles = (((B + 32) >> 5) + RPT - 1) / RPT;
    const int32_t nrows = ntiles * RPT;
    for (int32_t x = tid; x < nrows * 32; x += nthr) rowA[x] = 0;          // S_N = 0
    if (nwarps > 1) __syncthreads(); else __syncwarp();
    if (red[0]) {
        if (tid == 0) {
            P.best_gain[w] = 0;
            P.best_cost[w] = 0;
            P.feasible[w] = 0;
            atomic_min_i64(&P.status[1], w);
        }
        return;
    }
    const int32_t gtiles = (int32_t)(((Bb + 32) >> 5) + RPT - 1) / RPT;
    uint32_t *__restrict__ gch = reinterpret_cast<uint32_t *>(P.workspace + win->choice_offset);
    // !OSM: lane q K + k holds option k of the q-th frame of a chunk of CH = 32 / K frames, the next
    // chunk loaded while this one is consumed (as dp_window)
    const int CH = 32 / K;
    const int lq = lane / K, lk = lane - (lane / K) * K;
    int32_t a_gp = 0, a_c = 0, b_g = 0, b_c = 0;
    auto load_raw = [&](int32_t hi, int32_t &g, int32_t &c) {
        const int32_t i = hi - lq;
        g = 0;
        c = 0;
        if (lq < CH && i >= 0) load_opt(i, lk, g, c);
    };
    if (!OSM && N > 0) {
        int32_t g, c;
        load_raw(N - 1, g, c);
        a_gp = (g << 4) | (15 - lk);
        a_c = c;
        load_raw(N - 1 - CH, b_g, b_c);
    }
    int32_t *__restrict__ cur = rowA;
    int32_t *__restrict__ nxt = inplace ? rowA : rowB;
    const int32_t t0 = inplace ? ntiles - 1 : warp;
    const int32_t dt = inplace ? -1 : nwarps;
    const int32_t pad = P.pad_words;
    // rows of 32 cells that hold cells <= B: the last tile computes only its live rows, in groups of
    // four (rows above B are never read by a cell <= B; their choice bits are never walked). Short
    // rows are most of a mixed batch's windows (c5: B from 64) and a tile is 256 or 512 cells.
    const int32_t live_rows = (B + 32) >> 5;
    const int32_t last_groups = (live_rows - (ntiles - 1) * RPT + 3) >> 2;   // 1 .. RPT / 4
    // one tile: keys of its first NR rows from `cur`, values to `nxt`, choice word to the plane
    auto tile = [&](auto nr_tag, int32_t i, int32_t t, int q) {
        constexpr int NR = decltype(nr_tag)::value;
        const int32_t b_lo = t * RPT * 32;
        TCHECK(b_lo + RPT * 32 <= P.row_words && t < gtiles);
        int32_t key[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r) key[r] = NEG_R;
        for (int k = 0; k < K; ++k) {
            int32_t g, c;
            if (OSM) {
                const int2 v = opt_s[i * K + k];
                g = v.x;
                c = v.y;
            } else {
                g = __shfl_sync(0xffffffffu, a_gp, q * K + k);
                c = __shfl_sync(0xffffffffu, a_c, q * K + k);
            }
            if (c <= b_lo + pad) {
                TCHECK(b_lo - c >= -pad);
                const int32_t *__restrict__ s = cur + (b_lo + lane - c);
#pragma unroll
                for (int r = 0; r < NR; ++r) key[r] = max_plus(s[r * 32], g, key[r]);
            } else if (c < b_lo + NR * 32) {
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    const int32_t idx = b_lo + r * 32 + lane - c;
                    const int32_t v = idx < 0 ? NEG_R : cur[idx < 0 ? 0 : idx];
                    key[r] = max_plus(v, g, key[r]);
                }
            }
        }
        if (inplace) __syncwarp();                          // all reads of this tile done
        int32_t *__restrict__ dst = nxt + b_lo + lane;
#pragma unroll
        for (int r = 0; r < NR; ++r) dst[r * 32] = key[r] & ~15;
        gch[((int64_t)i * gtiles + t) * 32 + lane] = pack_choices<RPT, CB>(key);
    };
    int q = 0;                                              // frame index inside the option chunk
    for (int32_t i = N - 1; i >= 0; --i) {
        const int32_t f = N - 1 - i;
        if (!OSM && f > 0 && ++q == CH) {
            q = 0;
            a_gp = (b_g << 4) | (15 - lk);
            a_c = b_c;
            load_raw(i - CH, b_g, b_c);
        }
        for (int32_t t = t0; t >= 0 && t < ntiles; t += dt) {
            if (t < ntiles - 1 || last_groups * 4 >= RPT) {
                tile(std::integral_constant<int, RPT>(), i, t, q);
            } else if (CB == 4 || last_groups == 1) {       // RPT 8: 4 live rows; RPT 16: 4
                tile(std::integral_constant<int, 4>(), i, t, q);
            } else if (last_groups == 2) {
                tile(std::integral_constant<int, (CB == 2 ? 8 : 4)>(), i, t, q);
            } else {
                tile(std::integral_constant<int, (CB == 2 ? 12 : 4)>(), i, t, q);
            }
        }
        if (nwarps > 1) __syncthreads(); else __syncwarp();
        int32_t *tmp = cur;
        cur = nxt;
        nxt = tmp;
    }
    // ---- a4: G* = S_0[B], C* = min{b : S_0[b] = G*} (32-ary search by warp 0)
    const int32_t RB = cur[B];
    const bool feas = RB > VALID_MIN_R;
    const int32_t cnt = (warp == 0 && feas) ? warp_first_at_least(cur, B, RB, lane) : 0;
    if (tid == 0) {
        P.best_gain[w] = feas ? (RB >> 4) : (int32_t)red[1];
        P.best_cost[w] = feas ? cnt : (int32_t)red[2];
        P.feasible[w] = feas ? 1 : 0;
    }
}

// smem layout per CTA: [red: 8 x int64][pad][rowA][pad][rowB (G > 1)][options (OSM) | costs]
// [choice planes (solve smem)]. The pads (pad_words of -inf below each row buffer) are written
// once and never overwritten.
// U16 (NEXT-5, opt-in): fixed-K kernels that plan qualifying windows on u16 rows (dp_u16.cu).
// SMALL: launches of <= 4 warps per window (dp_small.cu): 72 registers instead of 64 (7 CTAs of
// 128 threads per SM), which removes the per-frame rematerialisation of loop invariants the
// 64-register budget forces (same-box A/B on c2: 40.9 -> 39.4 us per step).
template <int KSEL, int MODE, bool OSM, bool FUSE, bool U16 = false, bool SMALL = false>
// Register budget: 64 for fixed-K kernels (4 CTAs x 256 threads or 2 x 512 per SM); the
// mixed-K kernel inlines every K and gets 128 to avoid spilling its hot loop.
__global__ void __launch_bounds__(SMALL ? 128 : 512, SMALL ? 7 : ((KSEL == 0) ? 1 : 2)) dp_cta_kernel(DpParams P)
{
    extern __shared__ int4 smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    int64_t *red = reinterpret_cast<int64_t *>(smem_raw);
    int32_t *base = reinterpret_cast<int32_t *>(smem_raw) + 16;
    const int32_t stride = P.pad_words + P.row_words;
    int32_t *rowA = base + P.pad_words;
    int32_t *rowB = rowA + stride;
    int32_t *after = base + (nwarps > 1 ? 2 : 1) * stride;   // 16-B aligned (row_words % 32 == 0)
    int2 *opt_s = reinterpret_cast<int2 *>(after);
    int32_t *cst = after;                                      // !OSM: costs for the backtrack
    uint32_t *sch = reinterpret_cast<uint32_t *>(after + P.cst_words);
    __shared__ uint32_t hist[FUSE ? 176 : 1];
    for (int32_t x = threadIdx.x; x < P.pad_words; x += blockDim.x) {
        rowA[x - P.pad_words] = NEG_R;
        if (nwarps > 1) rowB[x - P.pad_words] = NEG_R;
    }
    __syncthreads();
    if (P.debug & 32) return;                         // timing: launch only
    if (KSEL == 0 && P.ordered) {
        // mixed-K kernel, serving order (the class's range of it): the window index comes from
        // memory, which is fine here -- the out-of-line bodies take it as a parameter anyway
        for (int64_t r = blockIdx.x; r < P.cls_count; r += gridDim.x) {
            const int64_t w = P.windows[P.cls_first + r].order;
            switch (P.windows[w].num_exits) {
#define TURBO_K_CASE(KK) \
    case KK: dp_window_call<KK, MODE, OSM, FUSE>(P, w, rowA, rowB, sch, cst, opt_s, red, hist, warp, nwarps, lane); \
        break;
                TURBO_K_CASE(2) TURBO_K_CASE(3) TURBO_K_CASE(4) TURBO_K_CASE(5) TURBO_K_CASE(6)
                TURBO_K_CASE(7) TURBO_K_CASE(8) TURBO_K_CASE(9) TURBO_K_CASE(10) TURBO_K_CASE(11)
                TURBO_K_CASE(12) TURBO_K_CASE(13) TURBO_K_CASE(14) TURBO_K_CASE(15) TURBO_K_CASE(16)
#undef TURBO_K_CASE
                default: break;
            }
            __syncthreads();                          // smem reused by the next window
            trace_mark(P, w, 5);
        }
        return;
    }
    // index order (fixed-K kernels always: their window index is the CTA index, which the
    // compiler keeps -- with the window's fields -- in uniform registers)
    for (int64_t w = blockIdx.x; w < P.num_windows; w += gridDim.x) {
        const int rc = row_class((int64_t)P.windows[w].budget_bound + 1);
        if (rc >= TURBO_NUM_CLASSES || (P.cls >= 0 && rc != P.cls)) continue;   // other launch serves it
        if (KSEL != 0) {
            dp_window<(KSEL > 0 ? KSEL : 2), MODE, OSM, FUSE, U16>(P, w, rowA, rowB, sch, cst, opt_s, red, hist,
                                                                  warp, nwarps, lane);
        } else {
            switch (P.windows[w].num_exits) {
#define TURBO_K_CASE(KK) \
    case KK: dp_window_call<KK, MODE, OSM, FUSE>(P, w, rowA, rowB, sch, cst, opt_s, red, hist, warp, nwarps, lane); \
        break;
                TURBO_K_CASE(2) TURBO_K_CASE(3) TURBO_K_CASE(4) TURBO_K_CASE(5) TURBO_K_CASE(6)
                TURBO_K_CASE(7) TURBO_K_CASE(8) TURBO_K_CASE(9) TURBO_K_CASE(10) TURBO_K_CASE(11)
                TURBO_K_CASE(12) TURBO_K_CASE(13) TURBO_K_CASE(14) TURBO_K_CASE(15) TURBO_K_CASE(16)
#undef TURBO_K_CASE
                default: break;
            }
        }
        __syncthreads();                              // smem reused by the next window
        trace_mark(P, w, 5);
    }
}

typedef void (*dp_kernel_t)(DpParams);

// Fixed-K specialisations for the exit counts of the paper-shaped workloads (beta = 3..7,
// PAPER.md:533 "4-5" levels, :919 beta = 5); any other K, and batches mixing K, run the
// mixed-K kernel (every K inlined behind a switch).
template <int MODE, bool OSM, bool FUSE = false>
dp_kernel_t pick_dp_kernel(int kmin, int kmax)
{
    if (!dp_kernel_fixed_k(kmin, kmax)) return dp_cta_kernel<0, MODE, OSM, FUSE>;
    switch (kmin) {
        case 4: return dp_cta_kernel<4, MODE, OSM, FUSE>;
        case 5: return dp_cta_kernel<5, MODE, OSM, FUSE>;
        case 6: return dp_cta_kernel<6, MODE, OSM, FUSE>;
        case 8: return dp_cta_kernel<8, MODE, OSM, FUSE>;
        default: return dp_cta_kernel<0, MODE, OSM, FUSE>;
    }
}

dp_kernel_t dp_kernel_plan(int kmin, int kmax, bool osm);
dp_kernel_t dp_kernel_generic(bool osm, bool fuse, bool small);
dp_kernel_t dp_kernel_solve_smem(int kmin, int kmax, bool osm);
dp_kernel_t dp_kernel_schedule(int kmin, int kmax, int mode, bool osm);
dp_kernel_t dp_kernel_u16(int kmin, int kmax, bool fuse);
dp_kernel_t dp_kernel_small(int kmin, int kmax, bool fuse);

}  // namespace turbo

// dp_pack.cu -- the MCKP DP for batches of short windows (c2-shaped: rows of a few tiles), V windows
// per CTA advanced in LOCKSTEP.
//
// Same recurrence, tie-break and outputs as dp_kernel.cuh (§5.2 with f = sum,
// readings R1, R7): frames N-1 .. 0, S_i[b] = max_{k : c_ik <= b} g_ik + S_{i+1}[b - c_ik], the
// smallest maximising k bit-packed per cell, G* = S_0[B], C* = #{b <= B : S_0[b] < G*}, forward walk.
//
// Why a second CTA kernel: with one CTA per window, a batch that fills the GPU in a single wave
// (c2: 1024 windows, 7 per SM) runs its windows as independent CTAs that the warp schedulers serve
// unevenly -- some finish early, and the last ones run alone on their SM, latency-bound, at the
// end (measured: DP phase 19.7 us median, 26.4 us max per window). Here one CTA holds V windows
// (their rows, option tables and choice planes all in shared memory) and its warps split the
// V x T tiles of a frame; ONE CTA barrier per frame advances every window together, so the SM's
// shared-memory pipe stays fed until the last frame and all V windows reach their epilogue
// together -- whose walks then run with the pipe otherwise idle.
//
// Layout per window slot v (words, stride P.pack_stride): [pad | rowA][pad | rowB][options int2
// N K][profile int2 C K (fused)][class ids u8 N (fused)][exits u8 N][choice planes N T 32].
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "dp_kernel.cuh"

namespace turbo {

struct PackWin {
    int64_t ff;
    int64_t g0, c0;                 // sums of option 0 (the infeasible report, reading R8)
    int32_t N, B, ntiles, bad;
    int32_t G, Cst, feas, prof;
};

constexpr int PACK_MAX_V = 32;

template <int K, bool FUSE>
__global__ void __launch_bounds__(1024, 1) dp_pack_kernel(DpParams P)
{
    constexpr int CB = (K <= 4) ? 2 : 4;
    constexpr int RPT = 32 / CB;
    extern __shared__ int4 smem_raw[];
    __shared__ PackWin ws[PACK_MAX_V];
    __shared__ uint32_t hist[FUSE ? 176 : 1];
    __shared__ unsigned long long tot[5];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int V = P.pack_v;
    const int64_t w0 = (int64_t)blockIdx.x * V;
    const int nv = (int)min((int64_t)V, (int64_t)P.num_windows - w0);
    const int32_t stride = P.pack_stride;
    const int32_t pad = P.pad_words, row = P.row_words;
    int32_t *const base = reinterpret_cast<int32_t *>(smem_raw);
    auto rowA = [&](int v) { return base + (int64_t)v * stride + pad; };
    auto rowB = [&](int v) { return base + (int64_t)v * stride + 2 * pad + row; };
    auto opts = [&](int v) { return reinterpret_cast<int2 *>(base + (int64_t)v * stride + 2 * (pad + row)); };
    auto profs = [&](int v) { return opts(v) + P.max_options; };
    auto clss = [&](int v) { return reinterpret_cast<uint8_t *>(profs(v) + P.prof_entries); };
    auto exs = [&](int v) { return clss(v) + ((P.max_frames + 3) & ~3); };
    auto planes = [&](int v) {
        return reinterpret_cast<uint32_t *>(exs(v) + ((P.max_frames + 3) & ~3));
    };

    // ---- prologue ----------------------------------------------------------------------------
    for (int v = 0; v < nv; ++v)
        for (int32_t x = tid; x < pad; x += nthr) {
            rowA(v)[x - pad] = NEG_R;
            rowB(v)[x - pad] = NEG_R;
        }
    if (FUSE) {
        for (int x = tid; x < 176; x += nthr) hist[x] = 0;
        if (tid < 5) tot[tid] = 0;
    }
    if (tid < nv) {                                          // per-window scalars (+ a1)
        const int64_t w = w0 + tid;
        const turbo_window_t win = P.windows[w];
        PackWin &s = ws[tid];
        s.ff = win.first_frame;
        s.N = win.num_frames;
        int32_t B = win.budget;
        if (FUSE && P.capacity != nullptr) {    // a1 (reading R3): max(0, capacity - m u0)
            const int64_t b = (int64_t)P.capacity[w] - (int64_t)win.num_frames * (int64_t)P.base_cost;
            B = (int32_t)(b < 0 ? 0 : (b > 0x7fffffffll ? 0x7fffffff : b));
            P.windows_rw[w].budget = B;
        }
        s.B = B;
        s.bad = (B < 0) || (B > win.budget_bound);
        s.ntiles = s.bad ? 0 : ((((B + 32) >> 5) + RPT - 1) / RPT);
        s.prof = win.profile;
        s.g0 = s.c0 = 0;
    }
    __syncthreads();
    if (FUSE) {
        // a2: class ids and the profile rows staged, then every option is
        // a shared-memory gather of its class's row (a class >= C gives a zero row + status[0])
        for (int v = 0; v < nv; ++v) {
            const turbo_profile_t &pr = P.profiles[ws[v].prof];
            const int32_t C = pr.num_classes;
            for (int32_t x = tid; x < ws[v].N; x += nthr) {
                const uint8_t c = (uint8_t)frame_class(P, ws[v].ff + x, C);
                clss(v)[x] = c;
                if (P.theta != nullptr) P.class_out[ws[v].ff + x] = c;      // NEXT-3 fused
            }
            for (int32_t x = tid; x < C * K; x += nthr) profs(v)[x] = make_int2(__ldg(pr.gain + x), __ldg(pr.cost + x));
        }
        __syncthreads();
    }
    for (int v = 0; v < nv; ++v) {
        const int32_t N = ws[v].N;
        bool bad = false;
        int2 *o = opts(v);
        if (FUSE) {
            const int32_t C = P.profiles[ws[v].prof].num_classes;
            for (int32_t q = tid; q < N * K; q += nthr) {
                const int32_t i = q / K, k = q - (q / K) * K;
                const int32_t cls = clss(v)[i];
                int32_t g = 0, c = 0;
                if (cls < C) {
                    const int2 pv = profs(v)[cls * K + k];
                    g = pv.x;
                    c = pv.y;
                } else if (k == 0) {
                    atomic_min_i64(&P.status[0], ws[v].ff + i);
                }
                bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
                o[q] = make_int2((g << 4) | (15 - k), c);
            }
        } else {
            const int32_t *og = P.opt_gain + P.windows[w0 + v].first_option;
            const int32_t *oc = P.opt_cost + P.windows[w0 + v].first_option;
            for (int32_t q = tid; q < N * K; q += nthr) {
                const int32_t g = __ldg(og + q), c = __ldg(oc + q);
                bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
                o[q] = make_int2((g << 4) | (15 - (q % K)), c);
            }
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&ws[v].bad, 1);
        // S_N = 0 on every cell of the row (whole tiles)
        const int32_t cells = ((((ws[v].B + 32) >> 5) + RPT - 1) / RPT) * RPT * 32;
        for (int32_t x = tid; x < cells && x < row; x += nthr) rowA(v)[x] = 0;
    }
    __syncthreads();
    if (warp < nv) {                                         // range rule + option-0 sums, warp v
        const int v = warp;
        const int2 *o = opts(v);
        int64_t abs_sum = 0, g0 = 0, c0 = 0;
        for (int32_t i = lane; i < ws[v].N; i += 32) {
            int32_t m = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int32_t g = o[i * K + k].x >> 4;
                m = max(m, g < 0 ? -g : g);
            }
            abs_sum += m;
            g0 += o[i * K].x >> 4;
            c0 += o[i * K].y;
        }
        abs_sum = warp_sum_i64(abs_sum);
        g0 = warp_sum_i64(g0);
        c0 = warp_sum_i64(c0);
        if (lane == 0) {
            ws[v].g0 = g0;
            ws[v].c0 = c0;
            if (abs_sum >= GAIN_RANGE_LIMIT || c0 >= 0x7fffffffll) ws[v].bad = 1;
        }
    }
    __syncthreads();

    // ---- a3: lockstep DP. Task q = v * T + t (window v, tile t); warp w takes q = w, w + G, ...
    const int T = P.pack_tiles;
    const int nq = nv * T;
    int32_t maxN = 0;
    for (int v = 0; v < nv; ++v) maxN = max(maxN, ws[v].bad ? 0 : ws[v].N);
    int32_t own[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) own[r] = 0;
    if (nq <= nwarps) {
        // one task per warp (the launch shape makes this the normal case): the task's addresses are
        // fixed for the whole window, the next frame's options are loaded before the barrier
        const int v = warp / T, t = warp - (warp / T) * T;
        const bool has = warp < nq && !ws[v].bad && t < ws[v].ntiles;
        const int32_t N = has ? ws[v].N : 0;
        const int32_t nt = has ? ws[v].ntiles : 1;
        const int32_t b_lo = t * RPT * 32;
        int32_t *const ra = rowA(has ? v : 0), *const rb = rowB(has ? v : 0);
        const int2 *const ov = opts(has ? v : 0);
        uint32_t *pl = planes(has ? v : 0) + ((int64_t)(N > 0 ? N - 1 : 0) * nt + t) * 32 + lane;
        int2 on[K];
        if (N > 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) on[k] = ov[(N - 1) * K + k];
        }
        for (int32_t f = 0; f < maxN; ++f) {
            if (f < N) {
                int32_t gp[K], cc[K];
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    gp[k] = on[k].x;
                    cc[k] = on[k].y;
                }
                if (f + 1 < N) {                             // frame i - 1's options, used after the barrier
#pragma unroll
                    for (int k = 0; k < K; ++k) on[k] = ov[(N - 2 - f) * K + k];
                }
                int32_t cmax = cc[0];
#pragma unroll
                for (int k = 1; k < K; ++k) cmax = max(cmax, cc[k]);
                const int32_t *cur = (f & 1) ? rb : ra;
                int32_t *nxt = (f & 1) ? ra : rb;
                TCHECK(b_lo + RPT * 32 <= row && (int64_t)(N - 1 - f) * nt * 32 + 32 <= P.chs_words);
                TCHECK(cmax > b_lo + pad || b_lo - cmax >= -pad);
                int32_t key[RPT];
                if (cmax <= b_lo + pad) {                    // every shift inside the -inf pad
                    const int32_t *src = cur + b_lo + lane;
                    if (cc[0] == 0) {
#pragma unroll
                        for (int r = 0; r < RPT; ++r) key[r] = own[r] + gp[0];
                    } else {
#pragma unroll
                        for (int r = 0; r < RPT; ++r) key[r] = src[r * 32 - cc[0]] + gp[0];
                    }
#pragma unroll
                    for (int k = 1; k < K; ++k) {
                        const int32_t *s = src - cc[k];
#pragma unroll
                        for (int r = 0; r < RPT; ++r) key[r] = max_plus(s[r * 32], gp[k], key[r]);
                    }
                } else {
                    tile_keys<K, RPT>(cur, b_lo, RPT, pad, gp, cc, lane, key);
                }
                int32_t *dst = nxt + b_lo + lane;
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const int32_t x = key[r] & ~15;
                    own[r] = x;
                    dst[r * 32] = x;
                }
                *pl = pack_choices<RPT, CB>(key);
                pl -= nt * 32;
            }
            __syncthreads();                                 // frame f of every window visible
        }
    } else {
        for (int32_t f = 0; f < maxN; ++f) {
            bool first = true;
            int v = warp / T, t = warp - (warp / T) * T;
            for (int q = warp; q < nq; q += nwarps) {
                const int32_t i = ws[v].N - 1 - f;
                const int32_t nt = ws[v].ntiles;
                if (i >= 0 && t < nt && !ws[v].bad) {
                    const int2 *o = opts(v) + i * K;
                    int32_t gp[K], cc[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const int2 x = o[k];
                        gp[k] = x.x;
                        cc[k] = x.y;
                    }
                    int32_t cmax = cc[0];
#pragma unroll
                    for (int k = 1; k < K; ++k) cmax = max(cmax, cc[k]);
                    const int32_t *cur = (f & 1) ? rowB(v) : rowA(v);
                    int32_t *nxt = (f & 1) ? rowA(v) : rowB(v);
                    if (first)
                        dp_tile<K, DP_SOLVE_SMEM, true>(P, t, i, nt * RPT, nt, 0, cur, nxt, planes(v), nullptr, gp,
                                                        cc, cmax, false, lane, own);
                    else
                        dp_tile<K, DP_SOLVE_SMEM, false>(P, t, i, nt * RPT, nt, 0, cur, nxt, planes(v), nullptr, gp,
                                                         cc, cmax, false, lane, own);
                }
                first = false;
                t += nwarps;                                 // next task: q + nwarps
                while (t >= T) {
                    t -= T;
                    ++v;
                }
            }
            __syncthreads();                                 // frame f of every window visible
        }
    }

    // ---- a4 / a5 / a6: warp v finishes window v (the pipe is idle now: walks run at latency)
    if (warp < nv) {
        const int v = warp;
        const int64_t w = w0 + v;
        PackWin &s = ws[v];
        const int32_t N = s.N, B = s.B;
        const int64_t ff = s.ff;
        uint8_t *ex_s = exs(v);
        if (s.bad) {
            if (lane == 0) {
                P.best_gain[w] = 0;
                P.best_cost[w] = 0;
                P.feasible[w] = 0;
                atomic_min_i64(&P.status[1], w);
            }
            for (int32_t i = lane; i < N; i += 32) {
                P.exit_out[ff + i] = 0;
                ex_s[i] = 0;
            }
            if (lane == 0) {
                s.G = 0;
                s.Cst = 0;
                s.feas = 0;
            }
        } else {
            const int32_t *S0 = (N & 1) ? rowB(v) : rowA(v);   // frame 0 was written at f = N - 1
            const int32_t RB = S0[B];
            const bool feas = RB > VALID_MIN_R;
            const int32_t cnt = feas ? warp_first_at_least(S0, B, RB, lane) : 0;
            const int32_t G = feas ? (RB >> 4) : (int32_t)s.g0;
            const int32_t Cst = feas ? cnt : (int32_t)s.c0;
            if (lane == 0) {
                P.best_gain[w] = G;
                P.best_cost[w] = Cst;
                P.feasible[w] = feas ? 1 : 0;
                s.G = G;
                s.Cst = Cst;
                s.feas = feas;
            }
            if (!feas) {
                for (int32_t i = lane; i < N; i += 32) {
                    P.exit_out[ff + i] = 0;
                    ex_s[i] = 0;
                }
            } else {
                const int2 *o = opts(v);
                auto cost = [&](int32_t i, int32_t k) -> int32_t { return o[i * K + k].y; };
                backtrack_warp<K, DP_SOLVE_SMEM>(N, Cst, planes(v), nullptr, s.ntiles, 0, cost, P.exit_out + ff,
                                                 ex_s, lane);
            }
        }
        __syncwarp();
        if (FUSE) {                                          // a6: CTA histogram + totals
            for (int32_t i = lane; i < N; i += 32) {
                const uint32_t k = ex_s[i];
                const uint32_t cls = clss(v)[i];
                atomicAdd(&hist[k], 1u);
                if (cls < 10) atomicAdd(&hist[16 + cls * 16 + k], 1u);
            }
            if (lane == 0) {
                atomicAdd(&tot[0], (unsigned long long)(long long)s.G);
                atomicAdd(&tot[1], (unsigned long long)(long long)s.Cst);
                atomicAdd(&tot[2], 1ull);
                atomicAdd(&tot[3], (unsigned long long)N);
                if (!s.feas) atomicAdd(&tot[4], 1ull);
            }
        }
    }
    if (FUSE) {
        __syncthreads();
        unsigned long long *st = reinterpret_cast<unsigned long long *>(P.stats);
        for (int x = tid; x < 176; x += nthr)
            if (hist[x]) atomicAdd(&st[x], (unsigned long long)hist[x]);
        if (tid < 5 && tot[tid]) atomicAdd(&st[176 + tid], tot[tid]);
    }
}

// ---------------------------------------------------------------------------------------------
// Host side: when the lockstep kernel serves a class, and its geometry.
static size_t pack_stride_words(const DpParams &P, int max_frames)
{
    const int64_t fr4 = (max_frames + 3) & ~3;
    return (size_t)(2 * (P.pad_words + P.row_words) + 2 * (int64_t)P.max_options + 2 * (int64_t)P.prof_entries +
                    fr4 / 4 + fr4 / 4 + P.chs_words);
}

typedef void (*pack_kernel_t)(DpParams);

static pack_kernel_t pick_pack(int K, bool fuse)
{
    switch (K) {
        case 4: return fuse ? dp_pack_kernel<4, true> : dp_pack_kernel<4, false>;
        case 5: return fuse ? dp_pack_kernel<5, true> : dp_pack_kernel<5, false>;
        case 6: return fuse ? dp_pack_kernel<6, true> : dp_pack_kernel<6, false>;
        case 8: return fuse ? dp_pack_kernel<8, true> : dp_pack_kernel<8, false>;
        default: return nullptr;
    }
}

// Geometry of a lockstep launch for a class shape: windows per CTA (V), tiles per window (T),
// warps, shared memory. Returns false when the class is not served by this kernel: K not one of
// the fixed-K instantiations, choice planes not in shared memory, too few windows per SM to gain
// anything, or a slot that does not fit.
bool pack_geometry(const turbo_shape_t *s, const DpParams &P, int num_sms, int smem_per_cta_max, int *V_out,
                   int *T_out, int *warps_out, size_t *smem_out)
{
    if (s->min_exits != s->max_exits || !pick_pack(s->max_exits, P.fuse != 0) || !P.osm || P.chs_words <= 0)
        return false;
    const int64_t W = s->num_windows;
    if (W < 2 * (int64_t)num_sms) return false;
    const int rpt = s->max_exits <= 4 ? 16 : 8;
    const int T = (int)((num_rows(s->max_budget_small) + rpt - 1) / rpt);
    if (T < 1 || T > 32) return false;
    const size_t stride = pack_stride_words(P, s->max_frames);
    const size_t stat = sizeof(PackWin) * PACK_MAX_V + 176 * 4 + 64 + 256;     // static smem (+ slack)
    if ((size_t)smem_per_cta_max <= stat) return false;
    const int v_smem = (int)(((size_t)smem_per_cta_max - stat) / (stride * 4));
    int V = (int)std::min<int64_t>(std::min<int64_t>(v_smem, 32 / T), PACK_MAX_V);
    V = (int)std::min<int64_t>(V, (W + num_sms - 1) / num_sms);
    if (V < 2) return false;
    *V_out = V;
    *T_out = T;
    *warps_out = V * T;
    *smem_out = stride * 4 * (size_t)V;
    return true;
}

cudaError_t launch_pack(const turbo_shape_t *s, const DpParams &P0, int num_sms, int smem_per_cta_max,
                        cudaStream_t stream)
{
    int V, T, warps;
    size_t smem;
    if (!pack_geometry(s, P0, num_sms, smem_per_cta_max, &V, &T, &warps, &smem)) return cudaErrorInvalidValue;
    DpParams P = P0;
    P.pack_v = V;
    P.pack_tiles = T;
    P.pack_stride = (int32_t)pack_stride_words(P, s->max_frames);
    P.max_frames = s->max_frames;
    pack_kernel_t kern = pick_pack(s->max_exits, P.fuse != 0);
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> limit;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        size_t &lim = limit[std::make_pair(dev, (const void *)kern)];
        if (smem > lim) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            lim = smem;
        }
    }
    const int64_t blocks = (s->num_windows + V - 1) / V;
    note_launch();
    kern<<<(unsigned)blocks, 32 * warps, smem, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace turbo

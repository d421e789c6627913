// dp_cluster.cu -- K4 for LARGE budgets: the MCKP DP of one window on one thread-block CLUSTER
// (the north star's "one CTA (or thread-block cluster for large budgets) per window").
//
// Same recurrence as dp_kernel.cuh (PAPER.md:519-525 with f = sum; readings R1, R7):
//     S_i[b] = max_{k : c_ik <= b} ( g_ik + S_{i+1}[b - c_ik] ),  frames N-1 .. 0.
// Rows longer than one CTA's shared memory (budget_bound + 1 > TURBO_BIG_CELLS) up to
// TURBO_CLUSTER_CELLS cells: CTA r of a cluster of CS (<= 16) owns the segment
// [r seg, (r + 1) seg) of the row in its shared memory for the whole window.
// A cell reads cells at or below itself: tiles whose reads stay inside the own segment use plain
// shared loads; the bottom tiles read the cells below the segment straight from the lower CTAs'
// shared memory through distributed shared memory (DSMEM: the cluster's shared windows mapped
// into the generic address space) -- no halo copy, no option-cost limit. The rows are TRIPLE-
// buffered and the cluster barrier is split (barrier.cluster.arrive.release at the end of a frame,
// wait.acquire inside the next): the tiles that neither read another segment nor hold cells a
// higher segment reads compute while the barrier completes; only the segment's bottom tiles
// (remote reads) and top tiles (read remotely) wait for it. Many long windows run
// at once, one per cluster, instead of one after another over the whole GPU (dp_grid.cu, which
// keeps the rows beyond TURBO_CLUSTER_CELLS, e.g. c4's 2^20). Choice planes go to HBM in the
// standard layout; a4 runs here, a5 (+ a6) in long_walk_kernel as for the grid path.
#include <cooperative_groups.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "dp_kernel.cuh"

namespace cg = cooperative_groups;

namespace turbo {

// 256 threads, fixed-K instantiations up to three CTAs per SM (85 registers, no spills) -- same box,
// 64 windows x 300 frames x 60,001 cells / 148 x 30,001 cells: 512 x 1 (128 registers) 4.62 / 8.53 ms,
// 512 x 2 (64 registers, spills) 3.03 / 6.47 ms, with the pushed halo 512 x 2 3.17 / 5.22, 384 x 2
// 2.52 / 4.75, 256 x 3 2.52 / 3.81 ms. The mixed-K instantiation: one CTA per SM.
constexpr int CL_THREADS = 256;
constexpr int CL_MINB_FIXED = 3;
constexpr int CL_MAX = 16;                 // largest cluster (8 portable, 16 with the opt-in)
constexpr int CL_NX = 5;                   // per-rank exchange words: bad, g0, c0, asum, cmax
constexpr int CL_HALO = 1024;              // cells below each segment buffer: the pushed halo
constexpr int CL_XCH = CL_MAX * CL_NX + 8; // exchange words (rank 0's copy is the cluster's)

__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__device__ __forceinline__ long long cl_block_sum(long long v, long long *sm, int tid, int nthr)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((tid & 31) == 0) sm[tid >> 5] = v;
    __syncthreads();
    long long s = 0;
    for (int x = 0; x < (nthr >> 5); ++x) s += sm[x];
    __syncthreads();
    return s;
}

// One window on the calling cluster. buf[m]: this CTA's three row buffers; base[m][q]: rank q's
// buffer m (generic DSMEM pointers).
template <int K>
__device__ __forceinline__ void cluster_window(const DpParams &P, cg::cluster_group &cluster, int64_t w, int32_t seg,
                                               int32_t lg_seg, int32_t *const *buf, int32_t *const (*base)[CL_MAX],
                                               long long *red, long long *xch0)
{
    constexpr int CB = (K <= 4) ? 2 : 4;
    constexpr int RPT = 32 / CB;
    constexpr int TC = 32 * RPT;                   // cells per tile
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
    const int rank = (int)cluster.block_rank(), CS = (int)cluster.num_blocks();

    const turbo_window_t *win = P.windows + w;
    const int64_t ff = win->first_frame;
    const int32_t N = win->num_frames;
    int32_t B = win->budget;
    const int32_t Bb = win->budget_bound;
    const int32_t *__restrict__ og = P.opt_gain + win->first_option;
    const int32_t *__restrict__ oc = P.opt_cost + win->first_option;
    // turbo_schedule (P.fuse): a1 budget from the capacity, a2 options straight from the frame's
    // class and the profile (a class >= C reads as a zero row and sets status[0], as the lookup)
    const bool fuse = P.fuse != 0;
    int32_t prof_C = 0;
    const int32_t *prof_g = nullptr, *prof_c = nullptr;
    if (fuse) {
        const turbo_profile_t *prof = P.profiles + win->profile;
        prof_C = prof->num_classes;
        prof_g = prof->gain;
        prof_c = prof->cost;
        if (P.capacity != nullptr) {       // a1 (reading R3): max(0, capacity - m u0)
            const int64_t b = (int64_t)P.capacity[w] - (int64_t)N * (int64_t)P.base_cost;
            B = (int32_t)(b < 0 ? 0 : (b > 0x7fffffffll ? 0x7fffffff : b));
            if (rank == 0 && tid == 0) P.windows_rw[w].budget = B;
        }
    }
    auto opt_g = [&](int32_t i, int32_t k) -> int32_t {
        if (!fuse) return __ldg(og + (int64_t)i * K + k);
        const int32_t cls = frame_class(P, ff + i, prof_C);
        return cls < prof_C ? __ldg(prof_g + cls * K + k) : 0;
    };
    auto opt_c = [&](int32_t i, int32_t k) -> int32_t {
        if (!fuse) return __ldg(oc + (int64_t)i * K + k);
        const int32_t cls = frame_class(P, ff + i, prof_C);
        return cls < prof_C ? __ldg(prof_c + cls * K + k) : 0;
    };
    uint32_t *__restrict__ gch = reinterpret_cast<uint32_t *>(P.workspace + win->choice_offset);
    const int32_t gtiles = (int32_t)(((Bb + 32) >> 5) + RPT - 1) / RPT;

    // ---- validation (range rule R14), class ids, and the infeasible-report sums, cluster-wide
    {
        long long bad = 0, g0 = 0, c0 = 0, asum = 0;
        int32_t cmx = 0;
        for (int32_t i = rank * nthr + tid; i < N; i += CS * nthr) {
            int32_t m = 0;
            if (fuse) {
                const int32_t cls = frame_class(P, ff + i, prof_C);
                if (cls >= prof_C) atomic_min_i64(&P.status[0], ff + i);
                if (P.theta != nullptr) P.class_out[ff + i] = (uint8_t)cls;    // NEXT-3 fused, for the walk
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int32_t g = opt_g(i, k);
                const int32_t c = opt_c(i, k);
                const int32_t a = g < 0 ? -g : g;
                m = a > m ? a : m;
                bad |= (c < 0) || (c >= (1 << 30)) || (g > (1 << 24)) || (g < -(1 << 24));
                cmx = max(cmx, c);
                if (k == 0) {
                    g0 += g;
                    c0 += c;
                }
            }
            asum += m;
        }
        bad = __syncthreads_or((int)bad);
        g0 = cl_block_sum(g0, red, tid, nthr);
        c0 = cl_block_sum(c0, red, tid, nthr);
        asum = cl_block_sum(asum, red, tid, nthr);
        cmx = __reduce_max_sync(0xffffffffu, (uint32_t)cmx);
        if (lane == 0) red[warp] = cmx;
        __syncthreads();
        if (tid == 0) {
            long long m = 0;
            for (int x = 0; x < nwarps; ++x) m = red[x] > m ? red[x] : m;
            xch0[rank * CL_NX + 0] = bad;
            xch0[rank * CL_NX + 1] = g0;
            xch0[rank * CL_NX + 2] = c0;
            xch0[rank * CL_NX + 3] = asum;
            xch0[rank * CL_NX + 4] = m;
        }
    }
    cluster.sync();
    if (tid == 0) {
        long long t[CL_NX] = {0, 0, 0, 0, 0};
        for (int q = 0; q < CS; ++q) {
            for (int x = 0; x < 4; ++x) t[x] += xch0[q * CL_NX + x];
            t[4] = xch0[q * CL_NX + 4] > t[4] ? xch0[q * CL_NX + 4] : t[4];
        }
        for (int x = 0; x < CL_NX; ++x) red[16 + x] = t[x];
    }
    __syncthreads();
    const long long g0_sum = red[16 + 1], c0_sum = red[16 + 2];
    const int32_t cmax_w = (int32_t)red[16 + 4];         // the window's largest option cost
    const bool bad = red[16] != 0 || red[16 + 3] >= GAIN_RANGE_LIMIT || c0_sum >= 0x7fffffffll || B < 0 || B > Bb;
    if (bad) {
        if (rank == 0 && tid == 0) {
            P.best_gain[w] = 0;
            P.best_cost[w] = 0;
            P.feasible[w] = 0;
            atomic_min_i64(&P.status[1], w);
        }
        cluster.sync();                            // the exchange words are reused by the next window
        return;
    }

    // ---- the own segment: tiles [t0, t0 + nt) of the row that hold cells <= B (whole tiles)
    const int32_t seg_lo = rank * seg;
    const int32_t live_tiles = (((B + 32) >> 5) + RPT - 1) / RPT;
    const int32_t t0 = seg_lo / TC;
    const int32_t nt = max(0, min(seg / TC, live_tiles - t0));
    TCHECK(seg % TC == 0 && (int64_t)CS * seg >= (int64_t)live_tiles * TC);
    for (int32_t x = tid; x < nt * TC; x += nthr) buf[0][x] = 0;         // S_N = 0 (buffer 0)
    // halos (CL_HALO cells below each buffer): rank 0's are -inf (cells below 0) for good; the
    // others hold the lower segment's top cells, pushed by its CTA as it computes them (S_N: 0)
    for (int32_t x = tid; x < CL_HALO; x += nthr) {
        buf[0][x - CL_HALO] = rank == 0 ? NEG_R : 0;
        if (rank == 0) {
            buf[1][x - CL_HALO] = NEG_R;
            buf[2][x - CL_HALO] = NEG_R;
        }
    }
    int32_t my_g = 0, my_c = 0;                    // lane k < K: option k of the next frame (raw)
    if (N > 0 && lane < K) {
        my_g = opt_g(N - 1, lane);
        my_c = opt_c(N - 1, lane);
    }
    __syncthreads();
    cl_arrive();                                   // phase "S_N written"

    const int32_t smask = seg - 1;
    const int32_t seg_hi = seg_lo + seg;
    // cells of the lower segment held locally: rank 0 its -inf pad, the others the pushed halo
    // (the top h_eff cells of the lower segment, h_eff = the window's largest cost, at most CL_HALO)
    const int32_t h_eff = min(CL_HALO, (cmax_w + 31) & ~31);
    const int32_t lo_local = seg_lo - (rank == 0 ? CL_HALO : h_eff);
    const bool push = rank + 1 < CS && h_eff > 0;
    int m = 0;                                     // buffer holding S_{i+1}; S_i goes to (m + 1) % 3
    int32_t key[RPT];
    for (int32_t f = 0; f < N; ++f) {
        const int32_t i = N - 1 - f;
        const int mw = m == 2 ? 0 : m + 1;
        const int32_t *cur = buf[m];
        int32_t *nxt = buf[mw];
        int32_t *const *cb = base[m];
        int32_t gp[K], cc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            gp[k] = (__shfl_sync(0xffffffffu, my_g, k) << 4) | (15 - k);
            cc[k] = __shfl_sync(0xffffffffu, my_c, k);
        }
        if (i > 0 && lane < K) {                   // consumed one frame later
            my_g = opt_g(i - 1, lane);
            my_c = opt_c(i - 1, lane);
        }
        int32_t cmax = cc[0];
#pragma unroll
        for (int k = 1; k < K; ++k) cmax = max(cmax, cc[k]);
        // a tile is SAFE when its reads stay in the own segment and no higher segment reads its
        // cells directly (the upper neighbour reads its pushed halo copy, unless the window has
        // costs beyond the halo): it may run before the barrier of the previous frame
        int32_t *nbh = push ? base[mw][rank + 1] : nullptr;     // upper neighbour's buffer (DSMEM)
        auto tile = [&](int32_t t) {
            const int32_t b_lo = t * TC;           // global cell of the tile's first row
            const int32_t lb = b_lo - seg_lo;      // its local index
            if (b_lo - cmax >= lo_local) {         // every read in the own segment or its halo
                tile_keys_fast<K, RPT>(cur + lane, lb, gp, cc, key);
            } else {
#pragma unroll
                for (int r = 0; r < RPT; ++r) key[r] = NEG_R;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const int32_t c = cc[k];
                    const int32_t x0 = b_lo - c;   // the option's first read
                    const int32_t q0 = x0 >> lg_seg, q1 = (x0 + TC - 1) >> lg_seg;
                    if (x0 >= lo_local) {          // own segment or halo
                        const int32_t *__restrict__ s = cur + (x0 - seg_lo) + lane;
#pragma unroll
                        for (int r = 0; r < RPT; ++r) key[r] = max_plus(s[r * 32], gp[k], key[r]);
                    } else if (x0 >= 0 && q0 == q1) {   // one lower segment: one base pointer
                        const int32_t *__restrict__ s = (q0 == rank ? cur : cb[q0]) + (x0 & smask) + lane;
#pragma unroll
                        for (int r = 0; r < RPT; ++r) key[r] = max_plus(s[r * 32], gp[k], key[r]);
                    } else {                       // straddles segments or cell 0: per cell
#pragma unroll
                        for (int r = 0; r < RPT; ++r) {
                            const int32_t x = x0 + r * 32 + lane;
                            TCHECK(x < 0 || (x >> lg_seg) <= rank);
                            const int32_t v = x < 0 ? NEG_R : cb[x >> lg_seg][x & smask];
                            key[r] = max_plus(v, gp[k], key[r]);
                        }
                    }
                }
            }
            int32_t *dst = nxt + lb + lane;
#pragma unroll
            for (int r = 0; r < RPT; ++r) dst[r * 32] = key[r] & ~15;
            TCHECK(t < gtiles);
            gch[((int64_t)i * gtiles + t) * 32 + lane] = pack_choices<RPT, CB>(key);
            if (push && b_lo + TC > seg_hi - h_eff) {    // top cells -> the upper neighbour's halo
                for (int r = 0; r < RPT; ++r) {          // (read back: key[] is dead by now)
                    const int32_t x = b_lo + r * 32 + lane;
                    if (x >= seg_hi - h_eff) nbh[x - seg_hi] = dst[r * 32];
                }
            }
        };
        // (the pushed halo of this frame is only complete after the barrier: a tile reading it is
        // not safe; rank 0's halo is the constant -inf pad)
        const int32_t safe_lo = rank == 0 ? lo_local : seg_lo;
        auto safe = [&](int32_t t) {
            return t * TC - cmax >= safe_lo && (cmax_w <= h_eff || t * TC + TC <= seg_hi - cmax_w);
        };
        __syncthreads();                           // the own S_{i+1} (previous frame) complete
        for (int32_t tl = warp; tl < nt; tl += nwarps)
            if (safe(t0 + tl)) tile(t0 + tl);
        cl_wait();                                 // every segment's S_{i+1} written, S_{i+2} read
        for (int32_t tl = warp; tl < nt; tl += nwarps)
            if (!safe(t0 + tl)) tile(t0 + tl);
        cl_arrive();
        m = mw;
    }
    cl_wait();                                     // S_0 complete cluster-wide
    const int32_t *cur = buf[m];
    int32_t *const *cb = base[m];

    // ---- a4: G* = S_0[B] (owner of B), C* = the first b <= B with S_0[b] >= G* (S_0 non-decreasing:
    // exactly one segment holds it -- the one whose last live cell reaches G* while the cell below
    // its first does not)
    if (rank == (B >> lg_seg) && tid == 0) xch0[CL_MAX * CL_NX] = cur[B - seg_lo];
    cluster.sync();
    if (tid == 0) red[16 + 5] = xch0[CL_MAX * CL_NX];
    __syncthreads();
    const int32_t RB = (int32_t)red[16 + 5];
    const bool feas = RB > VALID_MIN_R;
    if (feas && seg_lo <= B && warp == 0) {
        const int32_t last = min(seg_lo + seg - 1, B) - seg_lo;        // local index
        const bool reach = cur[last] >= RB;
        const bool below = rank == 0 || cb[rank - 1][seg - 1] < RB;    // cell seg_lo - 1 (DSMEM)
        if (reach && below) {
            const int32_t cnt = warp_first_at_least(cur, last, RB, lane);
            if (lane == 0) P.best_cost[w] = seg_lo + cnt;
        }
    }
    if (rank == 0 && tid == 0) {
        P.best_gain[w] = feas ? (RB >> 4) : (int32_t)g0_sum;
        if (!feas) P.best_cost[w] = (int32_t)c0_sum;
        P.feasible[w] = feas ? 1 : 0;
    }
    cluster.sync();                                // remote reads done before the buffers are reused
}

template <int K>
__device__ __noinline__ void cluster_window_call(const DpParams &P, cg::cluster_group &cluster, int64_t w, int32_t seg,
                                                 int32_t lg_seg, int32_t *const *buf, int32_t *const (*base)[CL_MAX],
                                                 long long *red, long long *xch0)
{
    cluster_window<K>(P, cluster, w, seg, lg_seg, buf, base, red, xch0);
}

// Cluster c serves the long windows r = c, c + clusters, ... (the serving order lists the long
// windows last, heaviest first); rows beyond `cap` cells are the grid kernel's.
template <int KSEL>
__global__ void __launch_bounds__(CL_THREADS, (KSEL == 0) ? 1 : CL_MINB_FIXED) dp_cluster_kernel(DpParams P, int32_t seg, int32_t lg_seg,
                                                                   int32_t cap, int32_t num_big)
{
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ int4 smem_raw[];
    long long *red = reinterpret_cast<long long *>(smem_raw);            // 16 scratch + 8 results
    long long *xch = red + 24;                                           // CL_XCH words
    int32_t *(*base)[CL_MAX] = reinterpret_cast<int32_t *(*)[CL_MAX]>(xch + CL_XCH);   // [3][CL_MAX]
    int32_t *buf[3];                               // [CL_HALO halo][seg cells] each
    buf[0] = reinterpret_cast<int32_t *>(base + 3) + CL_HALO;
    buf[1] = buf[0] + CL_HALO + seg;
    buf[2] = buf[1] + CL_HALO + seg;
    const int CS = (int)cluster.num_blocks();
    if (threadIdx.x < (unsigned)CS)
        for (int mm = 0; mm < 3; ++mm) base[mm][threadIdx.x] = cluster.map_shared_rank(buf[mm], (int)threadIdx.x);
    long long *xch0 = cluster.map_shared_rank(xch, 0);
    cluster.sync();                                // every block of the cluster is running
    const int64_t nclusters = gridDim.x / CS, cid = blockIdx.x / CS;
    const int64_t first = (int64_t)P.num_windows - num_big;
    for (int64_t r = cid; r < num_big; r += nclusters) {
        const int64_t w = P.ordered ? (int64_t)P.windows[first + r].order : r;
        const int64_t cells = (int64_t)P.windows[w].budget_bound + 1;
        if (cells <= TURBO_BIG_CELLS || cells > cap) continue;           // (uniform in the cluster)
        if (KSEL != 0) {
            cluster_window<(KSEL > 0 ? KSEL : 2)>(P, cluster, w, seg, lg_seg, buf, base, red, xch0);
        } else {
            switch (P.windows[w].num_exits) {
#define TURBO_K_CASE(KK) \
    case KK: cluster_window_call<KK>(P, cluster, w, seg, lg_seg, buf, base, red, xch0); break;
                TURBO_K_CASE(2) TURBO_K_CASE(3) TURBO_K_CASE(4) TURBO_K_CASE(5) TURBO_K_CASE(6)
                TURBO_K_CASE(7) TURBO_K_CASE(8) TURBO_K_CASE(9) TURBO_K_CASE(10) TURBO_K_CASE(11)
                TURBO_K_CASE(12) TURBO_K_CASE(13) TURBO_K_CASE(14) TURBO_K_CASE(15) TURBO_K_CASE(16)
#undef TURBO_K_CASE
                default: break;
            }
        }
    }
    cluster.sync();                                // no block leaves while another may read its smem
}

typedef void (*dp_cluster_kernel_t)(DpParams, int32_t, int32_t, int32_t, int32_t);

static dp_cluster_kernel_t pick_cluster(int kmin, int kmax)
{
    if (kmin == kmax) {
        switch (kmin) {
            case 4: return dp_cluster_kernel<4>;
            case 5: return dp_cluster_kernel<5>;
            case 6: return dp_cluster_kernel<6>;
            case 8: return dp_cluster_kernel<8>;
            default: break;
        }
    }
    return dp_cluster_kernel<0>;
}

// One candidate launch shape: segment seg (2^lg cells) and CS CTAs per cluster; sets the kernel's
// shared-memory (and, CS > 8, non-portable cluster size) attributes and asks for the resident
// clusters (cached per shape). cudaErrorInvalidConfiguration when no such cluster fits.
static cudaError_t try_geometry(dp_cluster_kernel_t kern, int32_t seg, int32_t lg, int CS, int smem_per_cta_max,
                                ClusterLaunch *out)
{
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)8 * (24 + CL_XCH + 3 * CL_MAX) + (size_t)12 * (seg + CL_HALO);
    if (smem + fa.sharedSizeBytes > (size_t)smem_per_cta_max) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // resident clusters: a host-side query, cached per (device, kernel, cluster size, smem)
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int, size_t>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, (const void *)kern, CS, smem);
    int nclusters = -1;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) nclusters = it->second;
    }
    if (nclusters < 0) {                // first use of this shape: the attributes, then the query
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess && CS > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&nclusters, (const void *)kern, &cfg);
        if (e != cudaSuccess) {
            cudaGetLastError();
            nclusters = 0;
        }
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = nclusters;
    }
    if (nclusters < 1) return cudaErrorInvalidConfiguration;
    out->kern = (const void *)kern;
    out->cs = CS;
    out->seg = seg;
    out->lg_seg = lg;
    out->smem = smem;
    out->max_clusters = nclusters;
    return cudaSuccess;
}

// Geometry of the cluster launch for the long windows of `shape` up to TURBO_CLUSTER_CELLS cells:
// rows up to 65,536 cells: a power-of-two segment >= 4,096 cells, CS = ceil(cells / seg) <= 8
// (portable); longer rows: 8,192-cell segments, 9..16 CTAs (non-portable cluster size, two CTAs
// per SM), else 16,384-cell segments, <= 8 CTAs (one CTA per SM: 16 x 120,001-cell windows 3.35 vs
// 2.5 ms). Shared memory incl. the static part and at least one resident cluster are checked here
// (host only), before any launch.
cudaError_t cluster_geometry(const turbo_shape_t *shape, int smem_per_cta_max, ClusterLaunch *out)
{
    const int64_t cells = std::min<int64_t>((int64_t)shape->max_budget + 1, TURBO_CLUSTER_CELLS);
    dp_cluster_kernel_t kern = pick_cluster(shape->min_exits, shape->max_exits);
    if (cells > 8 * 8192) {
        const int CS = (int)((cells + 8191) / 8192);
        if (try_geometry(kern, 8192, 13, CS, smem_per_cta_max, out) == cudaSuccess) return cudaSuccess;
    }
    int32_t seg = 4096, lg = 12;
    while ((int64_t)seg * 8 < cells) {
        seg *= 2;
        ++lg;
    }
    return try_geometry(kern, seg, lg, (int)((cells + seg - 1) / seg), smem_per_cta_max, out);
}

cudaError_t launch_dp_cluster(const turbo_shape_t *shape, const DpParams &P, int smem_per_cta_max, cudaStream_t stream)
{
    ClusterLaunch L;
    cudaError_t e = cluster_geometry(shape, smem_per_cta_max, &L);
    if (e != cudaSuccess) return e;
    // one cluster per long window (the block scheduler starts a cluster as soon as CS SMs free up;
    // capping the grid at a few waves of resident clusters made some clusters plan two windows
    // while the others idled: 64 windows on 60 clusters took twice the one-window time)
    const int64_t nclus = std::max<int64_t>(1, std::min<int64_t>(shape->num_big, (int64_t)(65535 / L.cs)));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = L.cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(nclus * L.cs));
    cfg.blockDim = dim3(CL_THREADS);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int32_t seg = L.seg, lg = L.lg_seg, cap = TURBO_CLUSTER_CELLS, nb = shape->num_big;
    note_launch();
    return cudaLaunchKernelEx(&cfg, (dp_cluster_kernel_t)L.kern, P, seg, lg, cap, nb);
}

}  // namespace turbo

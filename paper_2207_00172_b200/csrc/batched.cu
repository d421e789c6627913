// batched.cu -- NEXT-4: the exact plan under the paper's true, batched latency constraint.
//
// PAPER.md:523-525 (§5.2): maximise sum_x P_{kappa_x}^{theta'_x} s.t. f(sum I_kappa) <= T, with f
// batching the frames that run at the same level (a non-linear GAP). Latency does
// not depend on frame content, so a plan's cost depends only on its counts
// n_k = #{x : kappa_x = k}:  cost(n) = sum_k I_k(n_k)  (batch latency table, turbo.h).
// Readings: R19 -- gains have increasing differences in the class (PAPER.md:535-536,
// "the hardest frames have the largest marginals"), under which the assortative assignment
// (frames sorted by (class, arrival) fill level 0, then 1, ...) is an optimal transportation plan
// for its counts; so the optimum is a maximum over count vectors. R18 -- order: larger gain, then
// smaller cost, then the count vector read from the top level down lexicographically smaller,
// then that canonical assignment.
//
// B200 mapping: one CTA (256 threads) per window. The class histogram, the canonical positions
// and the per-level prefix gains P_k(j) (gain of the first j canonical frames at level k) are
// built in shared memory; then the C(N+K-1, K-1) count vectors are enumerated: each thread
// unranks prefixes (n_0 .. n_{K-3}) with a binomial table and sweeps the last two levels
// inline (cost and gain of a vector = 2K shared-memory reads, no global traffic); a 3-key
// (gain, cost, counts code) argmax reduces over the warp with shuffles and over the CTA in
// shared memory. Compute-bound on integer ALU + shared loads; tiny inputs, no HBM stream.
#include <algorithm>

#include "turbo_internal.cuh"

namespace turbo {

constexpr int BT_THREADS = 256;
constexpr int BT_MAX_N = 255;
constexpr int BT_MAX_K = 16;

struct BtParams {
    const turbo_window_t *windows;
    int32_t num_windows;
    int32_t general;             // 1: windows without R19 are left to batched_dp_kernel (R20);
                                 // 2: every valid window is (debug); 0: they are rejected
    const turbo_profile_t *profiles;
    const int32_t *batch;        // [profile][16][cap + 1]
    int32_t cap;
    const uint8_t *class_id;
    int32_t *best_gain;
    int32_t *best_cost;
    uint8_t *feasible;
    uint8_t *exit_out;
    int64_t *status;
};

// candidate order: larger gain, then smaller cost, then smaller counts code (R18)
__device__ __forceinline__ bool bt_better(int32_t g, int32_t c, uint64_t code, int32_t g2, int32_t c2,
                                          uint64_t code2)
{
    return g > g2 || (g == g2 && (c < c2 || (c == c2 && code < code2)));
}

// dynamic shared memory (kmax = the batch's largest K, cap = batch_cap):
//   pref  int32 [kmax][cap + 1]   P_k(j), gain of the first j canonical frames at level k
//   tab   int32 [kmax][cap + 1]   I_k(n)
//   binom u32   [cap + kmax + 1][kmax]  C(n, r), saturated at 2^31 (counts used stay < 2^26)
//   dif   int32 [cap + 1]         P_{K-2}(j) - P_{K-1}(j) (the inline sweep's gain term)
//   pos_cls u8  [cap]             class at canonical position j
__host__ __device__ inline size_t bt_smem_bytes(int32_t kmax, int32_t cap)
{
    return (size_t)2 * kmax * (cap + 1) * 4 + (size_t)(cap + kmax + 1) * kmax * 4 +
           (size_t)((cap + 1 + 3) & ~3) * 4 + (size_t)((cap + 15) & ~15);
}

__global__ void __launch_bounds__(BT_THREADS) batched_kernel(BtParams P, int32_t kmax)
{
    extern __shared__ int4 bt_dyn[];
    const int32_t ST = P.cap + 1;                           // row stride of pref / tab
    int32_t *pref_s = reinterpret_cast<int32_t *>(bt_dyn);
    int32_t *tab_s = pref_s + kmax * ST;
    uint32_t *binom_s = reinterpret_cast<uint32_t *>(tab_s + kmax * ST);
    int32_t *dif_s = reinterpret_cast<int32_t *>(binom_s + (P.cap + kmax + 1) * kmax);   // [cap + 1]
    uint8_t *pos_cls = reinterpret_cast<uint8_t *>(dif_s + ((P.cap + 1 + 3) & ~3));
#define pref(k, j) pref_s[(k) * ST + (j)]
#define tab(k, n) tab_s[(k) * ST + (n)]
#define binom(n, r) binom_s[(n) * kmax + (r)]
    __shared__ int32_t hist[257];
    __shared__ int32_t qsh[BT_MAX_K][257];                  // Q_k(c): gain of all smaller classes
    __shared__ int32_t red_g[BT_THREADS / 32], red_c[BT_THREADS / 32];
    __shared__ uint64_t red_k[BT_THREADS / 32];
    __shared__ int32_t flag;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int64_t w = blockIdx.x; w < P.num_windows; w += gridDim.x) {
        const turbo_window_t win = P.windows[w];
        const int32_t N = win.num_frames, B = win.budget;
        const turbo_profile_t pr = P.profiles[win.profile];
        const int32_t C = pr.num_classes, K = pr.num_exits;
        const uint8_t *cls = P.class_id + win.first_frame;
        const int32_t *gt = pr.gain;
        // ---- validation: class ids (status[0]), R19 and the budget (status[1])
        if (tid == 0) flag = 0;
        for (int x = tid; x < 257; x += BT_THREADS) hist[x] = 0;
        __syncthreads();
        for (int32_t x = tid; x < N; x += BT_THREADS) {
            const int32_t c = cls[x];
            if (c >= C) {
                atomic_min_i64(&P.status[0], win.first_frame + x);
                atomicOr(&flag, 1);
            } else {
                atomicAdd(&hist[c], 1);
            }
        }
        for (int32_t e = tid; e < (C - 1) * (K - 1); e += BT_THREADS) {
            const int32_t c = e / (K - 1), k = e - (e / (K - 1)) * (K - 1);
            const int64_t d1 = (int64_t)__ldg(gt + (c + 1) * K + k + 1) - __ldg(gt + (c + 1) * K + k);
            const int64_t d0 = (int64_t)__ldg(gt + c * K + k + 1) - __ldg(gt + c * K + k);
            if (d1 < d0) atomicOr(&flag, 2);
        }
        for (int32_t e = tid; e < C * K; e += BT_THREADS) {
            const int32_t v = __ldg(gt + e);
            if (v > (1 << 24) || v < -(1 << 24)) atomicOr(&flag, 2);
        }
        if (tid == 0 && (B < 0 || N > P.cap || N > BT_MAX_N)) atomicOr(&flag, 4);
        __syncthreads();
        // gains without R19 (flag 2 alone) go to the general program when it runs and can serve
        // the window (K <= 8, C <= 16; batched_dp_kernel)
        const bool dp_ok = K <= 8 && C <= 16;
        if (P.general == 2 && !(flag & 5) && dp_ok) continue;
        if (P.general == 1 && flag == 2 && dp_ok) continue;
        if (flag & 4) flag |= 2;
        if (flag) {
            if (tid == 0) {
                P.best_gain[w] = 0;
                P.best_cost[w] = 0;
                P.feasible[w] = 0;
                if (flag & 2) atomic_min_i64(&P.status[1], w);
            }
            for (int32_t x = tid; x < N; x += BT_THREADS) P.exit_out[win.first_frame + x] = 0;
            __syncthreads();
            continue;
        }
        // ---- canonical positions: class start offsets (exclusive prefix of the histogram)
        if (tid == 0) {
            int32_t s = 0;
            for (int32_t c = 0; c < C; ++c) {
                const int32_t m = hist[c];
                hist[c] = s;
                s += m;
            }
            hist[C] = s;
        }
        __syncthreads();
        for (int32_t j = tid; j < N; j += BT_THREADS) {             // class of position j
            int32_t c = 0;
            while (c + 1 < C && hist[c + 1] <= j) ++c;
            pos_cls[j] = (uint8_t)c;
        }
        // batch table rows and binomials C(n, r) (n <= N + K, r < K)
        const int32_t *bt = P.batch + (int64_t)win.profile * BT_MAX_K * (P.cap + 1);
        for (int32_t e = tid; e < K * (N + 1); e += BT_THREADS) {
            const int32_t k = e / (N + 1), n = e - (e / (N + 1)) * (N + 1);
            tab(k, n) = __ldg(bt + k * (P.cap + 1) + n);
        }
        for (int32_t n = tid; n <= N + K; n += BT_THREADS) {
            uint64_t v = 1;                                          // C(n, 0), exact while < 2^31
            for (int32_t r = 0; r < K; ++r) {
                binom(n, r) = r > n ? 0u : (uint32_t)(v < 0x80000000ull ? v : 0x80000000ull);
                if (v < 0x80000000ull) v = v * (uint64_t)(n - r) / (uint64_t)(r + 1);
            }
        }
        __syncthreads();
        // per-level prefix gains over the canonical order, P_k(j) = Q_k(c) + (j - start_c) g[c][k]
        // with c the class of position j-1 and Q_k(c) = sum_{c' < c} m_c' g[c'][k] (a short serial
        // pass over the classes per level, then every (k, j) in parallel)
        for (int32_t k = tid; k < K; k += BT_THREADS) {
            int64_t q = 0, qa = 0;
            for (int32_t c = 0; c < C; ++c) {
                qsh[k][c] = (int32_t)q;
                const int64_t gv = __ldg(gt + c * K + k);
                q += (int64_t)(hist[c + 1] - hist[c]) * gv;
                qa += (int64_t)(hist[c + 1] - hist[c]) * (gv < 0 ? -gv : gv);
            }
            if (qa > (1ll << 30)) atomicOr(&flag, 2);              // every partial sum fits int32
        }
        for (int32_t e = tid; e < K * (N + 1); e += BT_THREADS) {
            const int32_t t = tab(e / (N + 1), e - (e / (N + 1)) * (N + 1));
            if (t < 0 || t > (1 << 26)) atomicOr(&flag, 2);         // batch latencies (range)
        }
        __syncthreads();
        if (flag) {                                                 // range violation: rejected
            if (tid == 0) {
                P.best_gain[w] = 0;
                P.best_cost[w] = 0;
                P.feasible[w] = 0;
                atomic_min_i64(&P.status[1], w);
            }
            for (int32_t x = tid; x < N; x += BT_THREADS) P.exit_out[win.first_frame + x] = 0;
            __syncthreads();
            continue;
        }
        for (int32_t e = tid; e < K * (N + 1); e += BT_THREADS) {
            const int32_t k = e / (N + 1), j = e - (e / (N + 1)) * (N + 1);
            int32_t v = 0;
            if (j > 0) {
                const int32_t c = pos_cls[j - 1];
                v = qsh[k][c] + (j - hist[c]) * __ldg(gt + c * K + k);
            }
            pref(k, j) = v;
        }
        __syncthreads();
        for (int32_t j = tid; j <= N; j += BT_THREADS) dif_s[j] = pref(K - 2, j) - pref(K - 1, j);
        __syncthreads();

        // ---- enumerate the count vectors: prefixes (n_0 .. n_{K-3}) ranked lexicographically, the
        // last two levels swept inline. Each thread takes a contiguous range of prefix ranks: it
        // unranks its first prefix once (binomial search), then steps to the lexicographic
        // successor. (Measured alternatives: unranking every prefix, 285 us on b2; one vector per
        // step with per-lane carries, 361 us -- the carries diverge; this, 225 us.)
        const int32_t KP = K - 2;                                    // prefix parts
        const uint64_t n_pref = binom(N + KP, KP);                   // weak compositions, KP+1 parts
        int32_t bg = INT32_MIN, bc = INT32_MAX;
        uint64_t bk = ~0ull;
        const uint64_t chunk = (n_pref + BT_THREADS - 1) / BT_THREADS;
        const uint64_t r_lo = (uint64_t)tid * chunk;
        const uint64_t r_hi = r_lo + chunk < n_pref ? r_lo + chunk : n_pref;
        int32_t pv[BT_MAX_K];                                        // prefix parts n_0 .. n_{KP-1}
        int32_t left = N;                                            // the tail: n_{K-2} + n_{K-1}
        if (r_lo < r_hi) {
            uint64_t r = r_lo;
            for (int32_t i = 0; i < KP; ++i) {
                int32_t v = 0;
                for (;; ++v) {
                    // compositions of (left - v) into the remaining KP - i parts (incl. the tail)
                    const uint64_t cnt = binom(left - v + KP - i - 1, KP - i - 1);
                    if (r < cnt) break;
                    r -= cnt;
                }
                pv[i] = v;
                left -= v;
            }
        }
        for (uint64_t r0 = r_lo; r0 < r_hi; ++r0) {
            if (r0 > r_lo) {                                         // lexicographic successor
                if (left > 0) {
                    pv[KP - 1] += 1;
                    left -= 1;
                } else {
                    int32_t i = KP - 1;
                    while (i > 0 && pv[i] == 0) --i;                 // rightmost non-zero part
                    left += pv[i];
                    pv[i] = 0;
                    pv[i - 1] += 1;
                    left -= 1;
                }
            }
            int32_t S = 0, cost = 0, gain = 0;
            uint64_t code = 0, mul = 1;
            for (int32_t i = 0; i < KP; ++i) {
                const int32_t v = pv[i];
                cost += tab(i, v);
                gain += pref(i, S + v) - pref(i, S);
                if (i > 0) {                                         // n_0 is implied (sum = N)
                    code += (uint64_t)v * mul;
                    mul *= (uint64_t)(N + 1);
                }
                S += v;
            }
            // last two levels: n_{K-2} = v, n_{K-1} = left - v. Code weights: n_k counts
            // (N+1)^(k-1) for k >= 1 (n_0 is implied), so level K-2 weighs `mul` (0 when K = 2)
            const int32_t a2 = K - 2, b2 = K - 1;
            const uint64_t wa = a2 == 0 ? 0 : mul;
            const uint64_t wb = a2 == 0 ? 1 : mul * (uint64_t)(N + 1);
            const int32_t gb = gain + pref(b2, N) - pref(a2, S);
            // per vector: two batch-table reads, one read of the level-difference prefix gains, two
            // compares; the 64-bit counts code only when the vector is not worse than the best
            const int32_t *__restrict__ tA = &tab(a2, 0);
            const int32_t *__restrict__ tB = &tab(b2, left);          // tB[-v] = I_{K-1}(left - v)
            const int32_t *__restrict__ dd = dif_s + S;               // dd[v] = P_{K-2}(S+v) - P_{K-1}(S+v)
            for (int32_t v = 0; v <= left; ++v) {
                const int32_t c2 = cost + tA[v] + tB[-v];
                if (c2 > B) continue;
                const int32_t g2 = gb + dd[v];
                if (g2 < bg || (g2 == bg && c2 > bc)) continue;
                const uint64_t code2 = code + (uint64_t)v * wa + (uint64_t)(left - v) * wb;
                if (g2 > bg || c2 < bc || code2 < bk) {
                    bg = g2;
                    bc = c2;
                    bk = code2;
                }
            }
        }
        // ---- argmax over the CTA
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int32_t g2 = __shfl_xor_sync(0xffffffffu, bg, o);
            const int32_t c2 = __shfl_xor_sync(0xffffffffu, bc, o);
            const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bk, o);
            if (bt_better(g2, c2, k2, bg, bc, bk)) {
                bg = g2;
                bc = c2;
                bk = k2;
            }
        }
        if (lane == 0) {
            red_g[warp] = bg;
            red_c[warp] = bc;
            red_k[warp] = bk;
        }
        __syncthreads();
        if (tid == 0) {
            for (int x = 1; x < BT_THREADS / 32; ++x)
                if (bt_better(red_g[x], red_c[x], red_k[x], bg, bc, bk)) {
                    bg = red_g[x];
                    bc = red_c[x];
                    bk = red_k[x];
                }
            const bool feas = bk != ~0ull;
            const int32_t g0 = pref(0, N);
            P.best_gain[w] = feas ? bg : g0;
            P.best_cost[w] = feas ? bc : tab(0, N);
            P.feasible[w] = feas ? 1 : 0;
            // decode the counts into block boundaries S_k (reuse hist[0..K])
            int32_t rest = N, S = 0;
            uint64_t code = feas ? bk : 0;
            int32_t cnt[BT_MAX_K];
            for (int32_t k = 1; k < K; ++k) {
                cnt[k] = (int32_t)(code % (uint64_t)(N + 1));
                code /= (uint64_t)(N + 1);
                rest -= cnt[k];
            }
            cnt[0] = rest;
            for (int32_t k = 0; k < K; ++k) {                        // level blocks [S_k, S_k+1)
                hist[k] = S;
                S += cnt[k];
            }
            hist[K] = S;
        }
        __syncthreads();
        // ---- exits: frame x's canonical position -> its level block
        for (int32_t x = tid; x < N; x += BT_THREADS) {
            const int32_t c = cls[x];
            int32_t before = 0;                                      // same-class frames before x
            for (int32_t y = 0; y < x; ++y) before += (cls[y] == c) ? 1 : 0;
            int32_t start = 0;                                       // frames of smaller classes
            for (int32_t j = 0; j < N && pos_cls[j] < c; ++j) ++start;
            const int32_t posx = start + before;
            int32_t k = 0;
            while (k + 1 < K && hist[k + 1] <= posx) ++k;
            P.exit_out[win.first_frame + x] = (uint8_t)k;
        }
        __syncthreads();
    }
#undef pref
#undef tab
#undef binom
}

// ---------------------------------------------------------------------------------------------
// NEXT-4 for ANY gain table (reading R20; the windows whose gains lack R19). The gain of a count
// vector is then a C x K transportation optimum, computed for ALL count vectors at once by the
// program over the canonical prefix (frames sorted by (class, arrival)) and its count vector m:
//     F_0(0) = 0,   F_{j+1}(m) = max_{k : m_k > 0} F_j(m - e_k) + g[c_{x_j}][k],
// choice_{j+1}(m) = the HIGHEST maximising k (the backward walk then gives each frame the highest
// level that keeps the plan optimal -- R18's canonical plan whenever R19 holds). The count vector
// is chosen over the last layer exactly as batched_kernel does; the walk runs backwards from it.
// Layer j holds the C(j+K-1, K-1) compositions of j into K parts, ranked lexicographically; the
// ranks of the K predecessors m - e_k follow from m's rank terms by the hockey-stick identity in
// O(K) (no search). B200 mapping: one CTA per window at a time, the two F layers and the choice
// bytes of every layer in a per-CTA global scratch (L2-resident), threads sweep contiguous rank
// ranges of a layer (lexicographic successor), one CTA barrier per layer.
constexpr int BD_KMAX = 8;

__host__ __device__ inline int64_t bd_binom(int64_t n, int64_t r)
{
    if (r < 0 || n < r) return 0;
    int64_t v = 1;
    for (int64_t i = 0; i < r; ++i) v = v * (n - i) / (i + 1);
    return v;
}

// scratch per CTA (bytes): two int32 layers of the largest layer + the choice bytes of all layers
__host__ inline int64_t bd_scratch_bytes(int64_t N, int64_t K)
{
    const int64_t L = bd_binom(N + K - 1, K - 1);
    const int64_t T = bd_binom(N + K, K);
    return ((2 * 4 * L + T) + 255) & ~(int64_t)255;
}

__global__ void __launch_bounds__(BT_THREADS) batched_dp_kernel(BtParams P, uint8_t *scratch, int64_t per_cta,
                                                                 int32_t lmax)
{
    __shared__ int32_t hist[257];
    __shared__ int32_t order_s[BT_MAX_N + 1];                 // canonical position -> frame
    __shared__ uint8_t cls_pos[BT_MAX_N + 1];                 // canonical position -> class
    __shared__ int32_t gsh[16 * BD_KMAX];                     // gains of the window's profile (C <= 16)
    __shared__ uint32_t binom_s[BT_MAX_N + BD_KMAX + 2][BD_KMAX + 1];
    __shared__ int32_t red_g[BT_THREADS / 32], red_c[BT_THREADS / 32];
    __shared__ uint64_t red_k[BT_THREADS / 32];
    __shared__ int32_t flag;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int32_t *F0 = reinterpret_cast<int32_t *>(scratch + (int64_t)blockIdx.x * per_cta);
    int32_t *F1 = F0 + lmax;
    uint8_t *choice = reinterpret_cast<uint8_t *>(F1 + lmax);
    constexpr int32_t NEG = INT32_MIN / 2;

    for (int64_t w = blockIdx.x; w < P.num_windows; w += gridDim.x) {
        const turbo_window_t win = P.windows[w];
        const int32_t N = win.num_frames, B = win.budget;
        const turbo_profile_t pr = P.profiles[win.profile];
        const int32_t C = pr.num_classes, K = pr.num_exits;
        const uint8_t *cls = P.class_id + win.first_frame;
        const int32_t *gt = pr.gain;
        // the same validation as batched_kernel; this kernel takes the valid windows WITHOUT R19
        // (or every valid window, P.general == 2)
        if (tid == 0) flag = 0;
        for (int x = tid; x < 257; x += BT_THREADS) hist[x] = 0;
        __syncthreads();
        for (int32_t x = tid; x < N; x += BT_THREADS) {
            const int32_t c = cls[x];
            if (c >= C) atomicOr(&flag, 1); else atomicAdd(&hist[c], 1);
        }
        bool r19 = true;
        for (int32_t e = tid; e < (C - 1) * (K - 1); e += BT_THREADS) {
            const int32_t c = e / (K - 1), k = e - (e / (K - 1)) * (K - 1);
            const int64_t d1 = (int64_t)__ldg(gt + (c + 1) * K + k + 1) - __ldg(gt + (c + 1) * K + k);
            const int64_t d0 = (int64_t)__ldg(gt + c * K + k + 1) - __ldg(gt + c * K + k);
            if (d1 < d0) r19 = false;
        }
        if (!r19) atomicOr(&flag, 8);
        for (int32_t e = tid; e < C * K; e += BT_THREADS) {
            const int32_t v = __ldg(gt + e);
            if (v > (1 << 24) || v < -(1 << 24)) atomicOr(&flag, 2);
        }
        if (tid == 0 && (B < 0 || N > P.cap || N > BT_MAX_N || K > BD_KMAX || C > 16)) atomicOr(&flag, 4);
        __syncthreads();
        if (flag & 7) continue;                              // invalid: batched_kernel reports it
        if (P.general != 2 && !(flag & 8)) continue;         // R19 holds: batched_kernel plans it
        // canonical order and the class of each position
        if (tid == 0) {
            int32_t s = 0;
            for (int32_t c = 0; c < C; ++c) {
                const int32_t m = hist[c];
                hist[c] = s;
                s += m;
            }
            hist[C] = s;
        }
        for (int32_t e = tid; e < C * K; e += BT_THREADS) gsh[e] = __ldg(gt + e);
        for (int32_t n = tid; n <= N + K + 1; n += BT_THREADS)
            for (int32_t r = 0; r <= K; ++r) {
                const int64_t v = bd_binom(n, r);
                binom_s[n][r] = (uint32_t)(v < 0x7fffffffll ? v : 0x7fffffffll);
            }
        __syncthreads();
        if (tid == 0) {                                      // stable: arrival order inside a class
            for (int32_t x = 0; x < N; ++x) {
                const int32_t c = cls[x];
                const int32_t pos = hist[c]++;
                order_s[pos] = x;
                cls_pos[pos] = (uint8_t)c;
            }
        }
        // range rule of the partial sums (as batched_kernel): sum over frames of max |g| <= 2^30
        __syncthreads();
        if (tid == 0) {
            int64_t qa = 0;
            for (int32_t j = 0; j < N; ++j) {
                int64_t m = 0;
                for (int32_t k = 0; k < K; ++k) {
                    const int64_t v = gsh[cls_pos[j] * K + k];
                    m = max(m, v < 0 ? -v : v);
                }
                qa += m;
            }
            if (qa > (1ll << 30)) flag |= 2;
        }
        const int32_t *bt = P.batch + (int64_t)win.profile * BT_MAX_K * (P.cap + 1);
        for (int32_t e = tid; e < K * (N + 1); e += BT_THREADS) {
            const int32_t t = __ldg(bt + (e / (N + 1)) * (P.cap + 1) + e % (N + 1));
            if (t < 0 || t > (1 << 26)) atomicOr(&flag, 2);
        }
        __syncthreads();
        if (flag & 7) {                                      // range violation: rejected
            if (tid == 0) {
                P.best_gain[w] = 0;
                P.best_cost[w] = 0;
                P.feasible[w] = 0;
                atomic_min_i64(&P.status[1], w);
            }
            for (int32_t x = tid; x < N; x += BT_THREADS) P.exit_out[win.first_frame + x] = 0;
            __syncthreads();
            continue;
        }
        auto bn = [&](int32_t n, int32_t r) -> int64_t { return n < 0 ? 0 : (int64_t)binom_s[n][r]; };
        // ---- the program, layer by layer
        if (tid == 0) F0[0] = 0;
        int32_t *Fp = F0, *Fc = F1;
        int64_t choff = 0;                                   // choice bytes of layers 1 .. j
        __syncthreads();
        for (int32_t j = 1; j <= N; ++j) {
            const int32_t c = cls_pos[j - 1];
            const int64_t L = bn(j + K - 1, K - 1);
            const int64_t chunk = (L + BT_THREADS - 1) / BT_THREADS;
            const int64_t r_lo = (int64_t)tid * chunk, r_hi = min(r_lo + chunk, L);
            int32_t m[BD_KMAX];
#pragma unroll
            for (int k = 0; k < BD_KMAX; ++k) m[k] = 0;
            if (r_lo < r_hi) {                               // unrank the range's first composition
                int64_t r = r_lo;
                int32_t t = j;
#pragma unroll
                for (int i = 0; i < BD_KMAX - 1; ++i) {
                    if (i < K - 1) {
                        int32_t v = 0;
                        for (;; ++v) {
                            const int64_t cnt = bn(t - v + K - i - 2, K - i - 2);
                            if (r < cnt) break;
                            r -= cnt;
                        }
                        m[i] = v;
                        t -= v;
                    }
                }
#pragma unroll
                for (int i = 0; i < BD_KMAX; ++i)
                    if (i == K - 1) m[i] = t;
            }
            for (int64_t r = r_lo; r < r_hi; ++r) {
                if (r > r_lo) {                              // lexicographic successor
                    int32_t tail = 0, pos = -1;
#pragma unroll
                    for (int i = BD_KMAX - 1; i >= 0; --i) {
                        if (i < K) {
                            if (pos < 0 && i <= K - 2 && tail > 0) pos = i;
                            if (pos < 0) tail += m[i];
                        }
                    }
                    // increment m[pos], zero m[pos+1 .. K-2], m[K-1] = tail - 1
#pragma unroll
                    for (int i = 0; i < BD_KMAX; ++i) {
                        if (i == pos) m[i] += 1;
                        else if (i > pos && i < K - 1) m[i] = 0;
                        else if (i == K - 1) m[i] = tail - 1;
                    }
                }
                // rank terms: rank(m) = sum_{i <= K-2} A_i - B_i with t_0 = j, t_{i+1} = t_i - m_i,
                // A_i = C(t_i + K-i-1, K-i-1), B_i = C(t_{i+1} + K-i-1, K-i-1); for m - e_k the
                // terms i < k use t - 1 on both sides (Am, Bm), term k uses (Am_k, B_k)
                int64_t d[BD_KMAX], dm[BD_KMAX], am[BD_KMAX], bb[BD_KMAX];
                int32_t t = j;
#pragma unroll
                for (int i = 0; i < BD_KMAX - 1; ++i) {
                    d[i] = dm[i] = am[i] = bb[i] = 0;
                    if (i < K - 1) {
                        const int32_t p = K - i - 1, t1 = t - m[i];
                        const int64_t A = bn(t + p, p), Bv = bn(t1 + p, p);
                        const int64_t Am = bn(t - 1 + p, p), Bm = bn(t1 - 1 + p, p);
                        d[i] = A - Bv;
                        dm[i] = Am - Bm;
                        am[i] = Am;
                        bb[i] = Bv;
                        t = t1;
                    }
                }
                int64_t suffix = 0;                          // sum of d over i > k
#pragma unroll
                for (int i = 0; i < BD_KMAX - 1; ++i) suffix += d[i];
                int64_t prefix = 0;                          // sum of dm over i < k
                int32_t best = NEG, bk = 0;
#pragma unroll
                for (int k = 0; k < BD_KMAX; ++k) {
                    if (k < K) {
                        if (k < K - 1) suffix -= d[k];
                        if (m[k] > 0) {
                            const int64_t pr = prefix + (k < K - 1 ? am[k] - bb[k] : 0) + (k < K - 1 ? suffix : 0);
                            const int32_t prev = Fp[pr];
                            if (prev > NEG) {
                                const int32_t v = prev + gsh[c * K + k];
                                if (v >= best) {             // >=: the highest maximising level
                                    best = v;
                                    bk = k;
                                }
                            }
                        }
                        if (k < K - 1) prefix += dm[k];
                    }
                }
                Fc[r] = best;
                choice[choff + r] = (uint8_t)bk;
            }
            choff += L;
            __syncthreads();                                 // layer j complete
            int32_t *tmp = Fp;
            Fp = Fc;
            Fc = tmp;
        }
        // ---- the count vector: R18 order over the last layer (as batched_kernel)
        const int32_t *tab = bt;
        const int64_t L = bn(N + K - 1, K - 1);
        int32_t bg = INT32_MIN, bc = INT32_MAX;
        uint64_t bkey = ~0ull;
        {
            const int64_t chunk = (L + BT_THREADS - 1) / BT_THREADS;
            const int64_t r_lo = (int64_t)tid * chunk, r_hi = min(r_lo + chunk, L);
            for (int64_t r0 = r_lo; r0 < r_hi; ++r0) {
                // unrank (cheap enough for the last layer)
                int64_t r = r0;
                int32_t t = N, cost = 0;
                uint64_t code = 0, mul = 1;
                for (int32_t i = 0; i < K; ++i) {
                    int32_t v = t;
                    if (i < K - 1) {
                        v = 0;
                        for (;; ++v) {
                            const int64_t cnt = bn(t - v + K - i - 2, K - i - 2);
                            if (r < cnt) break;
                            r -= cnt;
                        }
                    }
                    cost += __ldg(tab + i * (P.cap + 1) + v);
                    if (i > 0) {
                        code += (uint64_t)v * mul;
                        mul *= (uint64_t)(N + 1);
                    }
                    t -= v;
                }
                const int32_t gain = Fp[r0];
                if (cost > B || gain <= NEG) continue;
                if (bt_better(gain, cost, code, bg, bc, bkey)) {
                    bg = gain;
                    bc = cost;
                    bkey = code;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int32_t g2 = __shfl_xor_sync(0xffffffffu, bg, o);
            const int32_t c2 = __shfl_xor_sync(0xffffffffu, bc, o);
            const uint64_t k2 = __shfl_xor_sync(0xffffffffu, bkey, o);
            if (bt_better(g2, c2, k2, bg, bc, bkey)) {
                bg = g2;
                bc = c2;
                bkey = k2;
            }
        }
        if (lane == 0) {
            red_g[warp] = bg;
            red_c[warp] = bc;
            red_k[warp] = bkey;
        }
        __syncthreads();
        if (tid == 0) {
            for (int x = 1; x < BT_THREADS / 32; ++x)
                if (bt_better(red_g[x], red_c[x], red_k[x], bg, bc, bkey)) {
                    bg = red_g[x];
                    bc = red_c[x];
                    bkey = red_k[x];
                }
            const bool feas = bkey != ~0ull;
            int64_t g0 = 0;
            for (int32_t x = 0; x < N; ++x) g0 += gsh[cls[x] * K];
            P.best_gain[w] = feas ? bg : (int32_t)g0;
            P.best_cost[w] = feas ? bc : __ldg(tab + N);
            P.feasible[w] = feas ? 1 : 0;
            if (!feas) {
                for (int32_t x = 0; x < N; ++x) P.exit_out[win.first_frame + x] = 0;
            } else {
                // backward walk: frame at canonical position j - 1 takes choice_j(m)
                int32_t m[16];
                uint64_t code = bkey;
                int32_t rest = N;
                for (int32_t k = 1; k < K; ++k) {
                    m[k] = (int32_t)(code % (uint64_t)(N + 1));
                    code /= (uint64_t)(N + 1);
                    rest -= m[k];
                }
                m[0] = rest;
                int64_t off = bn(N + K, K) - 1 - L;          // choice bytes before layer N
                for (int32_t j = N; j >= 1; --j) {
                    int64_t rk = 0;
                    int32_t t = j;
                    for (int32_t i = 0; i < K - 1; ++i) {
                        const int32_t p = K - i - 1;
                        rk += bn(t + p, p) - bn(t - m[i] + p, p);
                        t -= m[i];
                    }
                    const int32_t k = choice[off + rk];
                    P.exit_out[win.first_frame + order_s[j - 1]] = (uint8_t)k;
                    m[k] -= 1;
                    off -= bn(j - 1 + K - 1, K - 1);
                }
            }
        }
        __syncthreads();
    }
}

int64_t batched_dp_bytes(int32_t max_frames, int32_t max_exits, int num_sms)
{
    if (max_frames > BT_MAX_N) return 0;
    return (int64_t)num_sms * bd_scratch_bytes(max_frames, std::min(max_exits, BD_KMAX));
}

cudaError_t launch_batched(const turbo_window_t *windows, int32_t num_windows, const turbo_profile_t *profiles,
                           const int32_t *batch, int32_t cap, const uint8_t *class_id, int32_t *best_gain,
                           int32_t *best_cost, uint8_t *feasible, uint8_t *exit_out, int64_t *status, int32_t kmax,
                           int32_t max_frames, void *workspace, int32_t general, int num_sms, cudaStream_t stream)
{
    if (num_windows <= 0) return cudaSuccess;
    const size_t smem = bt_smem_bytes(kmax, cap);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    BtParams P;
    P.windows = windows;
    P.num_windows = num_windows;
    P.profiles = profiles;
    P.batch = batch;
    P.cap = cap;
    P.class_id = class_id;
    P.best_gain = best_gain;
    P.best_cost = best_cost;
    P.feasible = feasible;
    P.exit_out = exit_out;
    P.status = status;
    P.general = workspace != nullptr ? general : 0;
    int64_t blocks = num_windows;
    if (blocks > (int64_t)num_sms * 64) blocks = (int64_t)num_sms * 64;
    note_launch();
    batched_kernel<<<(unsigned)blocks, BT_THREADS, smem, stream>>>(P, kmax);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || workspace == nullptr) return e;
    // the windows without R19 (reading R20): one CTA per SM, per-CTA scratch in the workspace
    const int32_t kd = std::min(kmax, BD_KMAX);
    const int64_t per = bd_scratch_bytes(max_frames, kd);
    const int32_t lmax = (int32_t)bd_binom(max_frames + kd - 1, kd - 1);
    const int64_t dblocks = std::min<int64_t>(num_windows, num_sms);
    note_launch();
    batched_dp_kernel<<<(unsigned)dblocks, BT_THREADS, 0, stream>>>(P, reinterpret_cast<uint8_t *>(workspace), per,
                                                                    lmax);
    return cudaGetLastError();
}

}  // namespace turbo

/*
 * turbo_oracle.c -- CPU ORACLE for the Turbo enhancement-scheduler hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2207_00172_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant with it. Inputs come from synth/ (seeded generators).
 *
 * Plain, slow, obviously correct: int64 arithmetic, no blocking, no SIMD, one
 * thread per window (pthreads only ACROSS windows). Each function cites the
 * passage of /root/reference/PAPER.md (main paper, lines 164-997) it follows;
 * readings R1..R14 are listed in DESIGN.md.
 *
 * Parity pins (tests/test_oracle.py, -m "not gpu"): brute-force enumeration on
 * tiny windows (an independent pure-Python enumeration too), the worked instance
 * derived in SPEC.md:269 (tests/golden/), closed forms (unconstrained budget,
 * B = 0, K = 2 uniform-cost sort, K = 2 textbook 0/1 knapsack), invariants
 * (C* <= B, budget monotonicity PAPER.md:640, permutation invariance of G*).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <math.h>

#define ORACLE_NEG_INF INT64_MIN  /* "no plan of cost <= b exists" */

/* ------------------------------------------------------------------ a1: budget
 * PAPER.md:374 (§3) and :22 (draft A): the budget is set by "quantifying the
 * number of frames reaching the object detector". Reading R3:
 *   B_w = max(0, floor(T_w/q) - m_w * u0),  u0 = ceil(I_0/q),  I_0 = mu_D + nu_0
 * i.e. the idle GPU time left after the mandatory detection of the m_w frames. */
void oracle_budget(int32_t num_windows, const int32_t *capacity, const int32_t *num_frames,
                   int32_t base_cost, int32_t *budget_out)
{
    for (int32_t w = 0; w < num_windows; ++w) {
        int64_t b = (int64_t)capacity[w] - (int64_t)num_frames[w] * (int64_t)base_cost;
        budget_out[w] = (int32_t)(b < 0 ? 0 : b);
    }
}

/* ------------------------------------------------------------------ a2: lookup
 * PAPER.md:519-525 (§5.2): frame x with estimated difficulty theta'_x takes, for
 * level kappa, accuracy gain P_kappa^{theta'_x} (§5.1: profile per
 * bucket of width 0.1) and latency I_kappa. The per-frame
 * option table is therefore the profile row of the frame's class:
 *   opt_gain[x][k] = gain[class_x][k],  opt_cost[x][k] = cost[class_x][k].
 * Profiles are concatenated: profile p has C_p rows of K_p entries at prof_off[p].
 * Returns -1, or the smallest frame index whose class is out of range (its row is
 * then left zero). */
int64_t oracle_lookup(int32_t num_windows, const int32_t *num_frames, const int32_t *profile,
                      const uint8_t *class_id, const int32_t *prof_gain, const int32_t *prof_cost,
                      const int64_t *prof_off, const int32_t *prof_C, const int32_t *prof_K,
                      int32_t *opt_gain, int32_t *opt_cost)
{
    int64_t frame = 0, opt = 0, bad = -1;
    for (int32_t w = 0; w < num_windows; ++w) {
        int32_t p = profile[w], K = prof_K[p], C = prof_C[p];
        for (int32_t i = 0; i < num_frames[w]; ++i, ++frame) {
            int32_t cls = class_id[frame];
            for (int32_t k = 0; k < K; ++k, ++opt) {
                if (cls < C) {
                    opt_gain[opt] = prof_gain[prof_off[p] + (int64_t)cls * K + k];
                    opt_cost[opt] = prof_cost[prof_off[p] + (int64_t)cls * K + k];
                } else {
                    opt_gain[opt] = 0;
                    opt_cost[opt] = 0;
                    if (bad < 0) bad = frame;
                }
            }
        }
    }
    return bad;
}

/* ------------------------------------------------------------------ a3-a5: exact plan
 * The optimisation of PAPER.md:519-525 (§5.2, Eq. max / s.t.):
 *     max sum_x P_{kappa_x}^{theta'_x}   s.t.  f(sum I_kappa) <= T
 * with f = plain sum of per-frame incremental costs (reading R1: a multiple-choice
 * knapsack), computed EXACTLY, i.e. the paper's brute-force "upper" (PAPER.md:858,
 * §6.4). The result is the unique maximum of the total order (reading R7):
 *   (1) larger total gain, (2) then smaller total cost, (3) then the
 *   lexicographically smaller exit vector (frame 0 most significant).
 * No feasible plan (reading R8): all exits 0, gain = sum g_i0, cost = sum c_i0,
 * feasible = 0. Empty window: gain 0, cost 0, feasible. */

/* Brute force: enumerate all K^N plans in lexicographic order (frame N-1 fastest);
 * keep a plan only if strictly better in (gain, -cost), so the first one met among
 * equals -- the lexicographically smallest -- survives. */
int oracle_plan_brute(int32_t N, int32_t K, const int32_t *g, const int32_t *c, int32_t B,
                      uint8_t *exits, int64_t *best_gain, int64_t *best_cost, uint8_t *feasible)
{
    int32_t p[64];
    if (N > 64) return -1;
    int found = 0;
    int64_t bg = 0, bc = 0;
    for (int32_t i = 0; i < N; ++i) p[i] = 0;
    for (;;) {
        int64_t gain = 0, cost = 0;
        for (int32_t i = 0; i < N; ++i) {
            gain += g[(int64_t)i * K + p[i]];
            cost += c[(int64_t)i * K + p[i]];
        }
        if (cost <= B && (!found || gain > bg || (gain == bg && cost < bc))) {
            found = 1;
            bg = gain;
            bc = cost;
            for (int32_t i = 0; i < N; ++i) exits[i] = (uint8_t)p[i];
        }
        int32_t i = N - 1;                 /* odometer: last frame fastest */
        while (i >= 0 && ++p[i] == K) p[i--] = 0;
        if (i < 0) break;
    }
    if (!found) {
        bg = 0;
        bc = 0;
        for (int32_t i = 0; i < N; ++i) {
            exits[i] = 0;
            bg += g[(int64_t)i * K];
            bc += c[(int64_t)i * K];
        }
    }
    *best_gain = bg;
    *best_cost = bc;
    *feasible = (uint8_t)found;
    return 0;
}

/* Suffix table: T[i][b] = best gain of frames i..N-1 using total cost <= b
 * (-inf if none), T[N][b] = 0. G* = T[0][B]; C* = min{b : T[0][b] = G*};
 * forward reconstruction by value matching: at frame i with remaining budget r
 * and target value V take the smallest k with c_ik <= r and
 * g_ik + T[i+1][r - c_ik] = V. Table memory: (N+1)(B+1) int64. */
int oracle_plan_table(int32_t N, int32_t K, const int32_t *g, const int32_t *c, int32_t B,
                      uint8_t *exits, int64_t *best_gain, int64_t *best_cost, uint8_t *feasible)
{
    int64_t W = (int64_t)B + 1;
    int64_t *T = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1) * (size_t)W);
    if (!T) return -1;
    for (int64_t b = 0; b < W; ++b) T[(int64_t)N * W + b] = 0;
    for (int32_t i = N - 1; i >= 0; --i) {
        for (int64_t b = 0; b < W; ++b) {
            int64_t best = ORACLE_NEG_INF;
            for (int32_t k = 0; k < K; ++k) {
                int64_t ck = c[(int64_t)i * K + k];
                if (ck > b) continue;
                int64_t nxt = T[(int64_t)(i + 1) * W + (b - ck)];
                if (nxt == ORACLE_NEG_INF) continue;
                int64_t v = g[(int64_t)i * K + k] + nxt;
                if (v > best) best = v;
            }
            T[(int64_t)i * W + b] = best;
        }
    }
    int64_t G = T[B];
    if (G == ORACLE_NEG_INF) {
        int64_t bg = 0, bc = 0;
        for (int32_t i = 0; i < N; ++i) {
            exits[i] = 0;
            bg += g[(int64_t)i * K];
            bc += c[(int64_t)i * K];
        }
        *best_gain = bg;
        *best_cost = bc;
        *feasible = 0;
        free(T);
        return 0;
    }
    int64_t Cs = 0;
    while (T[Cs] != G) ++Cs;
    int64_t r = Cs, V = G;
    for (int32_t i = 0; i < N; ++i) {
        int32_t pick = -1;
        for (int32_t k = 0; k < K && pick < 0; ++k) {
            int64_t ck = c[(int64_t)i * K + k];
            if (ck > r) continue;
            int64_t nxt = T[(int64_t)(i + 1) * W + (r - ck)];
            if (nxt == ORACLE_NEG_INF) continue;
            if (g[(int64_t)i * K + k] + nxt == V) pick = k;
        }
        if (pick < 0) { free(T); return -2; }   /* cannot happen: table inconsistent */
        exits[i] = (uint8_t)pick;
        V -= g[(int64_t)i * K + pick];
        r -= c[(int64_t)i * K + pick];
    }
    *best_gain = G;
    *best_cost = Cs;
    *feasible = 1;
    free(T);
    return 0;
}

/* Value-only optimum for windows whose full table would not fit in memory:
 * the same recurrence over two rolling rows; returns G*, C*, feasibility. */
int oracle_optimum_rolling(int32_t N, int32_t K, const int32_t *g, const int32_t *c, int32_t B,
                           int64_t *best_gain, int64_t *best_cost, uint8_t *feasible)
{
    int64_t W = (int64_t)B + 1;
    int64_t *nxt = (int64_t *)malloc(sizeof(int64_t) * (size_t)W);
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)W);
    if (!nxt || !cur) { free(nxt); free(cur); return -1; }
    for (int64_t b = 0; b < W; ++b) nxt[b] = 0;
    for (int32_t i = N - 1; i >= 0; --i) {
        for (int64_t b = 0; b < W; ++b) {
            int64_t best = ORACLE_NEG_INF;
            for (int32_t k = 0; k < K; ++k) {
                int64_t ck = c[(int64_t)i * K + k];
                if (ck > b || nxt[b - ck] == ORACLE_NEG_INF) continue;
                int64_t v = g[(int64_t)i * K + k] + nxt[b - ck];
                if (v > best) best = v;
            }
            cur[b] = best;
        }
        int64_t *t = nxt; nxt = cur; cur = t;
    }
    int64_t G = nxt[B];
    if (G == ORACLE_NEG_INF) {
        int64_t bg = 0, bc = 0;
        for (int32_t i = 0; i < N; ++i) { bg += g[(int64_t)i * K]; bc += c[(int64_t)i * K]; }
        *best_gain = bg; *best_cost = bc; *feasible = 0;
    } else {
        int64_t Cs = 0;
        while (nxt[Cs] != G) ++Cs;
        *best_gain = G; *best_cost = Cs; *feasible = 1;
    }
    free(nxt); free(cur);
    return 0;
}

/* ------------------------------------------------------------------ batch driver
 * Windows are independent (one plan per window of m frames); the
 * driver only splits the window list across threads. mode: 0 = table, 1 = brute,
 * 2 = value-only (exits left untouched). */
typedef struct {
    int32_t num_windows, mode, nthreads, tid;
    const int32_t *num_frames, *budget, *K;
    const int64_t *first_frame, *first_option;
    const int32_t *opt_gain, *opt_cost;
    uint8_t *exits, *feasible;
    int64_t *best_gain, *best_cost;
    int err;
} oracle_job_t;

static void *oracle_worker(void *arg)
{
    oracle_job_t *j = (oracle_job_t *)arg;
    for (int32_t w = j->tid; w < j->num_windows; w += j->nthreads) {
        const int32_t *g = j->opt_gain + j->first_option[w];
        const int32_t *c = j->opt_cost + j->first_option[w];
        uint8_t *ex = j->exits ? j->exits + j->first_frame[w] : NULL;
        int r;
        if (j->mode == 1)
            r = oracle_plan_brute(j->num_frames[w], j->K[w], g, c, j->budget[w], ex,
                                  &j->best_gain[w], &j->best_cost[w], &j->feasible[w]);
        else if (j->mode == 2)
            r = oracle_optimum_rolling(j->num_frames[w], j->K[w], g, c, j->budget[w],
                                       &j->best_gain[w], &j->best_cost[w], &j->feasible[w]);
        else
            r = oracle_plan_table(j->num_frames[w], j->K[w], g, c, j->budget[w], ex,
                                  &j->best_gain[w], &j->best_cost[w], &j->feasible[w]);
        if (r) j->err = r;
    }
    return NULL;
}

int oracle_plan_batch(int32_t num_windows, const int32_t *num_frames, const int32_t *budget,
                      const int32_t *K, const int64_t *first_frame, const int64_t *first_option,
                      const int32_t *opt_gain, const int32_t *opt_cost, uint8_t *exits,
                      int64_t *best_gain, int64_t *best_cost, uint8_t *feasible,
                      int32_t mode, int32_t nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    oracle_job_t jobs[256];
    pthread_t th[256];
    for (int32_t t = 0; t < nthreads; ++t) {
        oracle_job_t j = {num_windows, mode, nthreads, t, num_frames, budget, K, first_frame,
                          first_option, opt_gain, opt_cost, exits, feasible, best_gain, best_cost, 0};
        jobs[t] = j;
    }
    if (nthreads == 1) {
        oracle_worker(&jobs[0]);
        return jobs[0].err;
    }
    for (int32_t t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, oracle_worker, &jobs[t]);
    int err = 0;
    for (int32_t t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].err) err = jobs[t].err;
    }
    return err;
}

/* ------------------------------------------------------------------ a6: statistics
 * Totals and histograms of the plans (the quantities PAPER.md §6 reports per run:
 * accuracy gain and enhancement usage), layout int64[181]:
 *   [0,16)    exits histogram (frames per chosen level kappa)
 *   [16,176)  class x exit histogram, classes 0..9 (PAPER.md:511 buckets), row-major
 *   176 sum of best_gain, 177 sum of best_cost, 178 #windows, 179 #frames,
 *   180 #infeasible windows. */
void oracle_stats(int32_t num_windows, const int32_t *num_frames, const uint8_t *class_id,
                  const uint8_t *exits, const int64_t *best_gain, const int64_t *best_cost,
                  const uint8_t *feasible, int64_t *stats)
{
    memset(stats, 0, sizeof(int64_t) * 181);
    int64_t f = 0;
    for (int32_t w = 0; w < num_windows; ++w) {
        for (int32_t i = 0; i < num_frames[w]; ++i, ++f) {
            int k = exits[f] & 15;
            stats[k] += 1;
            if (class_id[f] < 10) stats[16 + class_id[f] * 16 + k] += 1;
        }
        stats[176] += best_gain[w];
        stats[177] += best_cost[w];
        stats[178] += 1;
        stats[179] += num_frames[w];
        stats[180] += feasible[w] ? 0 : 1;
    }
}

/* ------------------------------------------------------------------ NEXT-1: the paper's heuristic
 * Prune-and-search, PAPER.md:539-545 (§5.2): "1) We assign all the m frames with the maximum
 * kappa. 2) ... we select the frame that has the minimal marginal accuracy gain, and assign
 * kappa-1. 3) We repeat the prior step until the T is met." With per-frame additive costs
 * (reading R1) the constraint is sum_i c_{i,k_i} <= B. Marginal gain of frame i at level k >= 1:
 * g_{i,k} - g_{i,k-1} (one-level difference). Ties: the larger
 * latency reduction c_{i,k} - c_{i,k-1} first, then the smaller frame id. Frames at level 0 cannot
 * be downgraded. If every frame reaches level 0 and the cost still exceeds B, the all-zero plan
 * is returned with feasible = 0. Returns the number of downgrade steps (<= N (K-1)). */
int64_t oracle_heuristic(int32_t N, int32_t K, const int32_t *g, const int32_t *c, int32_t B, uint8_t *exits,
                         int64_t *gain_out, int64_t *cost_out, uint8_t *feasible)
{
    int64_t cost = 0, steps = 0;
    for (int32_t i = 0; i < N; ++i) {
        exits[i] = (uint8_t)(K - 1);
        cost += c[(int64_t)i * K + K - 1];
    }
    while (cost > B) {
        int32_t pick = -1;
        int64_t best_m = 0, best_dc = 0;
        for (int32_t i = 0; i < N; ++i) {
            int32_t k = exits[i];
            if (k == 0) continue;
            int64_t m = (int64_t)g[(int64_t)i * K + k] - g[(int64_t)i * K + k - 1];
            int64_t dc = (int64_t)c[(int64_t)i * K + k] - c[(int64_t)i * K + k - 1];
            if (pick < 0 || m < best_m || (m == best_m && dc > best_dc)) {   /* smaller id wins: strict */
                pick = i;
                best_m = m;
                best_dc = dc;
            }
        }
        if (pick < 0) break;                /* everything at level 0 */
        exits[pick] -= 1;
        cost -= best_dc;
        steps += 1;
    }
    int64_t gain = 0;
    for (int32_t i = 0; i < N; ++i) gain += g[(int64_t)i * K + exits[i]];
    *gain_out = gain;
    *cost_out = cost;
    *feasible = (uint8_t)(cost <= B);
    return steps;
}

int oracle_heuristic_batch(int32_t num_windows, const int32_t *num_frames, const int32_t *budget, const int32_t *K,
                           const int64_t *first_frame, const int64_t *first_option, const int32_t *opt_gain,
                           const int32_t *opt_cost, uint8_t *exits, int64_t *gain, int64_t *cost, uint8_t *feasible,
                           int64_t *steps)
{
    for (int32_t w = 0; w < num_windows; ++w)
        steps[w] = oracle_heuristic(num_frames[w], K[w], opt_gain + first_option[w], opt_cost + first_option[w],
                                    budget[w], exits + first_frame[w], &gain[w], &cost[w], &feasible[w]);
    return 0;
}

/* ------------------------------------------------------------------ NEXT-3: score -> class
 * PAPER.md:511 (§5.1): frames are bucketised by difficulty with granularity 0.1; the online
 * classifier D_f gives the estimated score theta'_x. Reading R6: the class is the
 * bucket of d = 1 - theta' (class C-1 hardest); SPEC.md:65-73 bucket_index: floor(d / g), d = 1
 * clamped into the top bucket, d < 0 into bucket 0. The decision is taken in IEEE float32 (the
 * kernel's precision): d = 1 - theta (one rounding), q = d * (1/g) with 1/g given as a float32
 * (one rounding), class = floor(q) clamped to [0, C-1]. NaN scores map to class 0. */
void oracle_bucketize(int64_t n, const float *theta, float inv_width, int32_t C, uint8_t *cls)
{
    for (int64_t x = 0; x < n; ++x) {
        volatile float d = 1.0f - theta[x];
        volatile float q = d * inv_width;
        int32_t c = 0;
        if (q >= (float)C) c = C - 1;
        else if (q >= 0.0f) c = (int32_t)floorf(q);     /* NaN fails both tests -> 0 */
        if (c > C - 1) c = C - 1;
        cls[x] = (uint8_t)c;
    }
}

/* ------------------------------------------------------------------ NEXT-2: per-exit batches
 * PAPER.md:525 "organize the frames assigned by the same enhancement level to execute in a batch"
 * and :545 "we execute each frame according to the plan": per window, the frames of every exit
 * level kappa in arrival order (a stable partition), the batch sizes n_kappa, and the batch
 * offsets. Outputs: count[w*16 + k] = n_k; order[first_frame_w + j] = window-local frame index,
 * grouped by k ascending, arrival order within a group. */
void oracle_batches(int32_t num_windows, const int32_t *num_frames, const uint8_t *exits, int32_t *count,
                    int32_t *order)
{
    int64_t f0 = 0;
    for (int32_t w = 0; w < num_windows; ++w) {
        int32_t N = num_frames[w];
        for (int k = 0; k < 16; ++k) count[(int64_t)w * 16 + k] = 0;
        for (int32_t i = 0; i < N; ++i) count[(int64_t)w * 16 + exits[f0 + i]] += 1;
        int64_t pos = f0;
        for (int k = 0; k < 16; ++k)
            for (int32_t i = 0; i < N; ++i)
                if (exits[f0 + i] == k) order[pos++] = i;
        f0 += N;
    }
}

/* NEXT-2, executed latency (f "organize[s] the frames assigned by the same enhancement
 * level to execute in a batch"): f = sum over the levels k < K of I_k(n_k), the batch latency of the
 * n_k frames planned at level k (table I[k * (ncap + 1) + n]). A count above ncap: -1. */
void oracle_batch_latency(int32_t num_windows, const int32_t *count16, const int32_t *num_exits,
                          const int32_t *tables, const int64_t *table_off, const int32_t *profile, int32_t ncap,
                          int64_t *latency)
{
    for (int32_t w = 0; w < num_windows; ++w) {
        const int32_t *I = tables + table_off[profile[w]];
        int64_t f = 0;
        for (int32_t k = 0; k < num_exits[w]; ++k) {
            const int32_t n = count16[(int64_t)w * 16 + k];
            if (n > ncap) {
                f = -1;
                break;
            }
            f += I[(int64_t)k * (ncap + 1) + n];
        }
        latency[w] = f;
    }
}

/* ------------------------------------------------------------------ NEXT-4: batched-cost GAP
 * PAPER.md:523-525 (§5.2): maximise sum_x P_{kappa_x}^{theta'_x} subject to f(sum I_kappa) <= T,
 * where f batches the frames that run at the same level; PAPER.md:533 calls it a non-linear GAP.
 * Latency does not depend on frame content, so a plan's cost depends only on its
 * counts n_k = #{x : kappa_x = k}:   cost(n) = sum_k I_k(n_k),
 * with I_k(n) the batch latency of n frames at level k (table I[k * (ncap + 1) + n]).
 * Reading R18: the result is the unique maximum of -- larger gain, then smaller
 * cost, then the lexicographically smaller count vector read from the top level down
 * (n_{K-1}, ..., n_0), then the CANONICAL assignment for those counts: frames sorted by
 * (class, arrival index) fill level 0 first, then level 1, ... (contiguous blocks).
 * Reading R19: gains have increasing differences in the class ("the hardest
 * frames have the largest marginals"): g[c+1][k+1] - g[c+1][k] >= g[c][k+1] - g[c][k]. Then the
 * canonical assignment is optimal for its counts (assortative matching solves the C x K
 * transportation problem), so the optimum is a maximum over count vectors.
 * Infeasible (no count vector fits): all frames at level 0, feasible = 0, G = sum g[c_x][0],
 * C = I_0(N) (the analogue of reading R8).
 * Return: 0 ok; -1 bad arguments; -2 gains violate R19 (enum only). */

static int batched_r19_ok(int32_t C, int32_t K, const int32_t *g)
{
    for (int32_t c = 0; c + 1 < C; ++c)
        for (int32_t k = 0; k + 1 < K; ++k)
            if ((int64_t)g[(c + 1) * K + k + 1] - g[(c + 1) * K + k] < (int64_t)g[c * K + k + 1] - g[c * K + k])
                return 0;
    return 1;
}

/* canonical assignment of counts n[] to the N frames (see R18) */
static void batched_assign(int32_t N, int32_t C, int32_t K, const uint8_t *cls, const int32_t *n, uint8_t *exits)
{
    int32_t level = 0, left = n[0];
    for (int32_t c = 0; c < C; ++c)
        for (int32_t x = 0; x < N; ++x) {
            if ((int32_t)cls[x] != c) continue;
            while (left == 0 && level + 1 < K) left = n[++level];
            exits[x] = (uint8_t)level;
            left -= 1;
        }
    /* frames whose class is >= C never occur (validated by the caller) */
}

/* is count vector a lexicographically smaller than b, read from the top level down? */
static int batched_lex_less(int32_t K, const int32_t *a, const int32_t *b)
{
    for (int32_t k = K - 1; k >= 0; --k)
        if (a[k] != b[k]) return a[k] < b[k];
    return 0;
}

/* Brute force over all K^N plans (tiny N): the plain definition, no R19 needed for G*, C*;
 * best_counts = the lexicographically smallest count vector among the optimal plans. */
int oracle_batched_brute(int32_t N, int32_t C, int32_t K, const uint8_t *cls, const int32_t *g,
                         const int32_t *I, int32_t ncap, int32_t B, int64_t *best_gain, int64_t *best_cost,
                         int32_t *best_counts, uint8_t *feasible)
{
    if (N < 0 || N > 12 || K < 2 || K > 16 || N > ncap) return -1;
    int64_t total = 1;
    for (int32_t i = 0; i < N; ++i) total *= K;
    int32_t plan[16], cnt[16];
    int have = 0;
    int64_t bg = 0, bc = 0;
    int32_t bn[16];
    for (int64_t code = 0; code < total; ++code) {
        int64_t r = code;
        for (int32_t k = 0; k < K; ++k) cnt[k] = 0;
        int64_t gain = 0;
        for (int32_t i = 0; i < N; ++i) {
            plan[i] = (int32_t)(r % K);
            r /= K;
            cnt[plan[i]] += 1;
            gain += g[(int32_t)cls[i] * K + plan[i]];
        }
        int64_t cost = 0;
        for (int32_t k = 0; k < K; ++k) cost += I[k * (ncap + 1) + cnt[k]];
        if (cost > B) continue;
        int better = !have || gain > bg || (gain == bg && cost < bc) ||
                     (gain == bg && cost == bc && batched_lex_less(K, cnt, bn));
        if (better) {
            have = 1;
            bg = gain;
            bc = cost;
            for (int32_t k = 0; k < K; ++k) bn[k] = cnt[k];
        }
    }
    if (!have) {
        int64_t g0 = 0;
        for (int32_t i = 0; i < N; ++i) g0 += g[(int32_t)cls[i] * K];
        for (int32_t k = 0; k < K; ++k) bn[k] = k == 0 ? N : 0;
        bg = g0;
        bc = I[N];
    }
    *best_gain = bg;
    *best_cost = bc;
    *feasible = (uint8_t)have;
    for (int32_t k = 0; k < K; ++k) best_counts[k] = bn[k];
    return 0;
}

/* recursive enumeration of the compositions n_0 + ... + n_{K-1} = N */
typedef struct {
    int32_t N, C, K, ncap, B;
    const int32_t *I;
    const int64_t *P;            /* P[k * (N + 1) + j]: gain of the first j sorted frames at level k */
    int32_t n[16], bn[16];
    int have;
    int64_t bg, bc;
} batched_ctx;

static void batched_rec(batched_ctx *x, int32_t k, int32_t left)
{
    if (k == x->K - 1) {
        x->n[k] = left;
        int64_t cost = 0, gain = 0;
        int32_t s = 0;
        for (int32_t j = 0; j < x->K; ++j) {
            cost += x->I[j * (x->ncap + 1) + x->n[j]];
            gain += x->P[j * (x->N + 1) + s + x->n[j]] - x->P[j * (x->N + 1) + s];
            s += x->n[j];
        }
        if (cost > x->B) return;
        int better = !x->have || gain > x->bg || (gain == x->bg && cost < x->bc) ||
                     (gain == x->bg && cost == x->bc && batched_lex_less(x->K, x->n, x->bn));
        if (better) {
            x->have = 1;
            x->bg = gain;
            x->bc = cost;
            for (int32_t j = 0; j < x->K; ++j) x->bn[j] = x->n[j];
        }
        return;
    }
    for (int32_t v = 0; v <= left; ++v) {
        x->n[k] = v;
        batched_rec(x, k + 1, left - v);
    }
}

/* Exact optimum by count-vector enumeration (R18, R19): one window. */
int oracle_batched_enum(int32_t N, int32_t C, int32_t K, const uint8_t *cls, const int32_t *g, const int32_t *I,
                        int32_t ncap, int32_t B, uint8_t *exits, int64_t *best_gain, int64_t *best_cost,
                        uint8_t *feasible)
{
    if (N < 0 || K < 2 || K > 16 || C < 1 || N > ncap) return -1;
    if (!batched_r19_ok(C, K, g)) return -2;
    for (int32_t i = 0; i < N; ++i)
        if ((int32_t)cls[i] >= C) return -1;
    /* frames in canonical order (class, arrival) and the per-level prefix gains */
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    int64_t *P = (int64_t *)malloc(sizeof(int64_t) * (size_t)K * (size_t)(N + 1));
    int32_t t = 0;
    for (int32_t c = 0; c < C; ++c)
        for (int32_t i = 0; i < N; ++i)
            if ((int32_t)cls[i] == c) order[t++] = i;
    for (int32_t k = 0; k < K; ++k) {
        P[k * (N + 1)] = 0;
        for (int32_t j = 0; j < N; ++j) P[k * (N + 1) + j + 1] = P[k * (N + 1) + j] + g[(int32_t)cls[order[j]] * K + k];
    }
    batched_ctx x;
    memset(&x, 0, sizeof(x));
    x.N = N;
    x.C = C;
    x.K = K;
    x.ncap = ncap;
    x.B = B;
    x.I = I;
    x.P = P;
    batched_rec(&x, 0, N);
    if (!x.have) {
        int64_t g0 = 0;
        for (int32_t i = 0; i < N; ++i) g0 += g[(int32_t)cls[i] * K];
        for (int32_t k = 0; k < K; ++k) x.bn[k] = k == 0 ? N : 0;
        x.bg = g0;
        x.bc = I[N];
    }
    batched_assign(N, C, K, cls, x.bn, exits);
    *best_gain = x.bg;
    *best_cost = x.bc;
    *feasible = (uint8_t)x.have;
    free(order);
    free(P);
    return 0;
}

/* windows of a batch (one table pair per window via profile index) */
/* ------------------------------------------------------------------ NEXT-4 for ANY gain table
 * Reading R20: without R19 the canonical assignment need not be optimal for its counts,
 * so the gain of a count vector n is the transportation optimum
 *     gain(n) = max { sum_x g[c_x][kappa_x] : #{x : kappa_x = k} = n_k for every k }.
 * The count vector is chosen as in R18 (larger gain, then smaller cost, then (n_{K-1}, .., n_0)
 * lexicographically smaller). The assignment: frames in canonical order (class, then arrival)
 * x_0 .. x_{N-1}; going BACKWARDS from x_{N-1}, each frame takes the highest level k that still
 * admits an optimal completion. (Under R19 this is R18's canonical assignment: the canonical plan is
 * optimal, and its last frame sits on the highest used level.)
 *
 * Plain algorithm: dynamic program over the canonical prefix x_0 .. x_{j-1} and the count vector m
 * of that prefix (total j):  F_0(0) = 0,
 *     F_{j+1}(m) = max over k with m_k > 0 of F_j(m - e_k) + g[c_{x_j}][k],
 * so F_N(n) = gain(n). Count vectors are stored in a dense mixed-radix table (index
 * sum_{k>=1} m_k (N+1)^(k-1); m_0 is implied by the total) -- small windows only (tests).
 * Return: 0 ok; -1 bad arguments or table too large. */
static int64_t bdp_index(int32_t K, int32_t N, const int32_t *m)
{
    int64_t idx = 0, mul = 1;
    for (int32_t k = 1; k < K; ++k) {
        idx += (int64_t)m[k] * mul;
        mul *= (N + 1);
    }
    return idx;
}

int oracle_batched_dp(int32_t N, int32_t C, int32_t K, const uint8_t *cls, const int32_t *g, const int32_t *I,
                      int32_t ncap, int32_t B, uint8_t *exits, int64_t *best_gain, int64_t *best_cost,
                      uint8_t *feasible)
{
    if (N < 0 || K < 2 || K > 16 || C < 1 || N > ncap) return -1;
    int64_t S = 1;                               /* (N+1)^(K-1) table entries per prefix length */
    for (int32_t k = 1; k < K; ++k) {
        S *= (N + 1);
        if (S > (1ll << 24)) return -1;
    }
    for (int32_t i = 0; i < N; ++i)
        if ((int32_t)cls[i] >= C) return -1;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    int32_t t = 0;
    for (int32_t c = 0; c < C; ++c)
        for (int32_t i = 0; i < N; ++i)
            if ((int32_t)cls[i] == c) order[t++] = i;
    const int64_t NEG = INT64_MIN / 4;
    int64_t *F = (int64_t *)malloc(sizeof(int64_t) * (size_t)(N + 1) * (size_t)S);   /* F[j][index] */
    for (int64_t e = 0; e < (int64_t)(N + 1) * S; ++e) F[e] = NEG;
    F[0] = 0;
    int32_t m[16];
    for (int32_t j = 0; j < N; ++j) {
        const int32_t c = cls[order[j]];
        /* every count vector of total j + 1: iterate the table, keep entries whose total fits */
        for (int64_t idx = 0; idx < S; ++idx) {
            int64_t r = idx;
            int32_t tot = 0;
            for (int32_t k = 1; k < K; ++k) {
                m[k] = (int32_t)(r % (N + 1));
                r /= (N + 1);
                tot += m[k];
            }
            if (tot > j + 1) continue;
            m[0] = j + 1 - tot;
            int64_t best = NEG;
            for (int32_t k = 0; k < K; ++k) {
                if (m[k] == 0) continue;
                m[k] -= 1;
                const int64_t prev = F[(int64_t)j * S + bdp_index(K, N, m)];
                m[k] += 1;
                if (prev == NEG) continue;
                const int64_t v = prev + g[c * K + k];
                if (v > best) best = v;
            }
            F[(int64_t)(j + 1) * S + idx] = best;
        }
    }
    /* choose the count vector (R18 order over the final layer) */
    int have = 0;
    int64_t bg = 0, bc = 0;
    int32_t bn[16];
    for (int64_t idx = 0; idx < S; ++idx) {
        int64_t r = idx;
        int32_t tot = 0;
        for (int32_t k = 1; k < K; ++k) {
            m[k] = (int32_t)(r % (N + 1));
            r /= (N + 1);
            tot += m[k];
        }
        if (tot > N) continue;
        m[0] = N - tot;
        const int64_t gain = F[(int64_t)N * S + idx];
        if (gain == NEG) continue;
        int64_t cost = 0;
        for (int32_t k = 0; k < K; ++k) cost += I[k * (ncap + 1) + m[k]];
        if (cost > B) continue;
        int better = !have || gain > bg || (gain == bg && cost < bc) ||
                     (gain == bg && cost == bc && batched_lex_less(K, m, bn));
        if (better) {
            have = 1;
            bg = gain;
            bc = cost;
            for (int32_t k = 0; k < K; ++k) bn[k] = m[k];
        }
    }
    if (!have) {
        int64_t g0 = 0;
        for (int32_t i = 0; i < N; ++i) g0 += g[(int32_t)cls[i] * K];
        for (int32_t i = 0; i < N; ++i) exits[i] = 0;
        *best_gain = g0;
        *best_cost = I[N];
        *feasible = 0;
    } else {
        /* backwards: frame x_{j-1} takes the highest level that keeps F optimal */
        for (int32_t k = 0; k < K; ++k) m[k] = bn[k];
        for (int32_t j = N; j >= 1; --j) {
            const int32_t c = cls[order[j - 1]];
            const int64_t target = F[(int64_t)j * S + bdp_index(K, N, m)];
            int32_t pick = -1;
            for (int32_t k = K - 1; k >= 0 && pick < 0; --k) {
                if (m[k] == 0) continue;
                m[k] -= 1;
                const int64_t prev = F[(int64_t)(j - 1) * S + bdp_index(K, N, m)];
                m[k] += 1;
                if (prev != NEG && prev + g[c * K + k] == target) pick = k;
            }
            exits[order[j - 1]] = (uint8_t)pick;
            m[pick] -= 1;
        }
        *best_gain = bg;
        *best_cost = bc;
        *feasible = 1;
    }
    free(F);
    free(order);
    return 0;
}

/* The R20 assignment by its definition, for tiny windows: among all K^N plans with the optimal
 * gain, cost and count vector (brute force), the one whose exits read in REVERSE canonical order
 * (x_{N-1} first) are lexicographically largest. */
int oracle_batched_brute_plan(int32_t N, int32_t C, int32_t K, const uint8_t *cls, const int32_t *g,
                              const int32_t *I, int32_t ncap, int32_t B, uint8_t *exits, int64_t *best_gain,
                              int64_t *best_cost, uint8_t *feasible)
{
    int32_t bn[16];
    int e = oracle_batched_brute(N, C, K, cls, g, I, ncap, B, best_gain, best_cost, bn, feasible);
    if (e) return e;
    if (!*feasible) {
        for (int32_t i = 0; i < N; ++i) exits[i] = 0;
        return 0;
    }
    int32_t order[16], t = 0;
    for (int32_t c = 0; c < C; ++c)
        for (int32_t i = 0; i < N; ++i)
            if ((int32_t)cls[i] == c) order[t++] = i;
    int64_t total = 1;
    for (int32_t i = 0; i < N; ++i) total *= K;
    int32_t plan[16], cnt[16], best[16];
    int have = 0;
    for (int64_t code = 0; code < total; ++code) {
        int64_t r = code;
        for (int32_t k = 0; k < K; ++k) cnt[k] = 0;
        int64_t gain = 0;
        for (int32_t i = 0; i < N; ++i) {
            plan[i] = (int32_t)(r % K);
            r /= K;
            cnt[plan[i]] += 1;
            gain += g[(int32_t)cls[i] * K + plan[i]];
        }
        int same = gain == *best_gain;
        for (int32_t k = 0; k < K && same; ++k) same = cnt[k] == bn[k];
        if (!same) continue;
        int larger = !have;
        for (int32_t j = N - 1; j >= 0 && !larger; --j) {
            const int32_t a = plan[order[j]], b = best[order[j]];
            if (a != b) {
                larger = a > b;
                break;
            }
        }
        if (larger) {
            have = 1;
            for (int32_t i = 0; i < N; ++i) best[i] = plan[i];
        }
    }
    for (int32_t i = 0; i < N; ++i) exits[i] = (uint8_t)best[i];
    return 0;
}

int oracle_batched_batch(int32_t num_windows, const int32_t *num_frames, const int32_t *budget,
                         const int32_t *profile, const int64_t *first_frame, const uint8_t *class_id,
                         const int32_t *gains, const int64_t *gain_off, const int32_t *C, const int32_t *K,
                         const int32_t *batch, const int64_t *batch_off, int32_t ncap, uint8_t *exits,
                         int64_t *best_gain, int64_t *best_cost, uint8_t *feasible)
{
    for (int32_t w = 0; w < num_windows; ++w) {
        const int32_t p = profile[w];
        int e = oracle_batched_enum(num_frames[w], C[p], K[p], class_id + first_frame[w], gains + gain_off[p],
                                    batch + batch_off[p], ncap, budget[w], exits + first_frame[w], &best_gain[w],
                                    &best_cost[w], &feasible[w]);
        if (e == -2)                /* gains without R19: the general program (reading R20) */
            e = oracle_batched_dp(num_frames[w], C[p], K[p], class_id + first_frame[w], gains + gain_off[p],
                                  batch + batch_off[p], ncap, budget[w], exits + first_frame[w], &best_gain[w],
                                  &best_cost[w], &feasible[w]);
        if (e) return e;
    }
    return 0;
}

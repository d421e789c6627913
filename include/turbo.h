/*
 * turbo.h -- C ABI of the B200 (sm_100a) hot path of Turbo's online enhancement
 * scheduler (arXiv 2207.00172, "Turbo: Opportunistic Enhancement for Edge Video
 * Analytics", §5 Adaptive Enhancement Scheduling).
 *
 * Problem (§5.2, Eq. max / s.t.): a window holds m frames x
 * with estimated difficulty theta'_x (a class = bucket of width 0.1);
 * choose an enhancement level kappa_x in [0, beta] for every frame to maximise
 * sum_x P_{kappa_x}^{theta'_x} subject to the window's latency constraint T.
 * With per-frame additive costs (reading R1 in DESIGN.md) this is a multiple-choice
 * knapsack, solved EXACTLY (the paper's brute-force "upper") by an
 * integer max-plus dynamic program. Result = unique maximum of the total order
 * (gain desc, cost asc, exit vector lexicographically asc, frame 0 first).
 *
 * Conventions for every entry point:
 *  - Pointers are DEVICE pointers unless marked (host). Device buffers are owned by
 *    the caller and must stay alive until the stream work completes; the library
 *    keeps no reference after a call returns and never allocates device memory.
 *  - Calls are stream-ordered on `stream` (a cudaStream_t; NULL = legacy default
 *    stream), never synchronise the device, and are re-entrant / thread-safe.
 *  - Host-side validation runs before any launch; on error nothing is launched and
 *    the status code says why. Launch failures return TURBO_ERR_CUDA.
 *  - Integer units: gains in 0.01 mAP points (|g| <= 2^24), costs in GPU-time units
 *    (0 <= c < 2^31), budgets in the same units. Gains of one window must satisfy
 *    sum_i max_k |g_ik| < 2^25 (range rule R14) -- checked on device per window.
 */
#ifndef TURBO_H
#define TURBO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TURBO_OK = 0,
    TURBO_ERR_INVALID_ARG = 1,   /* null pointer, bad count, K outside [2,16], C outside [1,256] */
    TURBO_ERR_RANGE = 2,         /* N_w > 65535, budget outside [0, 2^30), sizes overflow        */
    TURBO_ERR_WORKSPACE = 3,     /* workspace smaller than turbo_mckp_workspace() demanded       */
    TURBO_ERR_CUDA = 4,          /* a kernel launch or attribute query failed                    */
    TURBO_ERR_UNSUPPORTED = 5    /* shape the compiled kernels cannot serve (e.g. row > smem)   */
} turbo_status_t;

typedef void *turbo_stream_t;    /* cudaStream_t */

/* One offline profile (§5.1): accuracy gain P_kappa^theta per
 * difficulty bucket and level, and latency cost I_kappa per level, both quantised.
 * Row-major [class][exit]; exit 0 = "no enhancement" (P_0 = 0 in the paper, not
 * required here). Costs are INCREMENTAL over mandatory detection (reading R3). */
typedef struct {
    int32_t num_classes;         /* C in [1, 256]                                   */
    int32_t num_exits;           /* K = beta + 1 in [2, 16]                         */
    const int32_t *gain;         /* device [C*K]                                    */
    const int32_t *cost;         /* device [C*K], >= 0                              */
} turbo_profile_t;

/* One scheduling window: the m_w frames reaching the detector and its budget. */
typedef struct {
    int64_t first_frame;         /* offset into class_id[] / exit_out[] (caller sets)            */
    int64_t first_option;        /* offset into opt_gain[] / opt_cost[] (turbo_mckp_workspace)   */
    int64_t choice_offset;       /* byte offset of this window's choice plane in the workspace  */
    int32_t num_frames;          /* m_w in [0, 65535] (caller sets)                              */
    int32_t budget;              /* B_w >= 0 (caller sets, or a1 derives it on device)           */
    int32_t profile;             /* index into the profile array (caller sets)                   */
    int32_t num_exits;           /* K of the profile (turbo_mckp_workspace)                      */
    int32_t budget_bound;        /* layout bound: budget at sizing time (turbo_mckp_workspace);
                                    a device-side budget above it rejects the window            */
    int32_t order;               /* (turbo_mckp_workspace) a permutation stored across the
                                    array: order of entry r = the window served r-th -- windows
                                    grouped by row-size class, largest work N (B+1) (K+1) first
                                    inside a class (longest-processing-time first)             */
} turbo_window_t;                /* 48 bytes; array lives on the host (sizing) and the device */

/* Launch shape of a window batch, computed on the host by turbo_mckp_workspace
 * from the host copies of windows and profiles. Passed (host) to every device
 * call so the library never reads device memory to configure a launch. */
typedef struct {
    int32_t num_windows;
    int32_t num_profiles;
    int32_t max_frames;          /* max m_w                                      */
    int32_t max_budget;          /* max budget_bound                              */
    int32_t min_exits, max_exits;
    int32_t num_classes_max;
    int32_t max_options;         /* max over windows of m_w K_w (one window's option table)  */
    int64_t total_frames;        /* sum m_w                                       */
    int64_t total_options;       /* sum m_w K_w  (size of opt_gain / opt_cost)    */
    int64_t total_cells;         /* sum m_w (budget_bound_w + 1)                  */
    int64_t workspace_bytes;     /* bytes needed by turbo_mckp_plan / backtrack   */
    int32_t max_budget_small;    /* max budget_bound over windows served by one CTA each        */
    int32_t num_big;             /* windows whose row (budget_bound + 1 > TURBO_BIG_CELLS cells)
                                    is split over the whole grid (long-window kernel)           */
    int64_t grid_scratch_offset; /* workspace offset of the long-window kernel's halo ring/flags */
    int32_t ordered;             /* 1: the kernels serve windows through turbo_window_t.order
                                    (several classes, or uneven work); 0: in index order        */
    int32_t cls_order;           /* launch order of the row-size classes, 4 bits each from the
                                    lowest nibble (turbo_mckp_workspace: 0x0123, longest rows
                                    first); not a permutation -> 0x3210                   */
    int64_t reserved3;
    /* per row-size class (TURBO_NUM_CLASSES, see below): windows of one class are planned by one
     * launch shaped for them (warps per window, shared memory, residency) */
    int32_t cls_count[4];
    int32_t cls_max_budget[4];
    int32_t cls_max_frames[4];
    int32_t cls_max_options[4];
    int32_t cls_min_exits[4];
    int32_t cls_max_exits[4];
} turbo_shape_t;

/* Row-size classes of windows served by one CTA each: class c holds the windows with
 * budget_bound + 1 <= TURBO_CLASS_CELLS_c cells (and above the previous bound). */
#define TURBO_NUM_CLASSES 4
#define TURBO_CLASS_CELLS_0 256
#define TURBO_CLASS_CELLS_1 1024
#define TURBO_CLASS_CELLS_2 4608
#define TURBO_CLASS_CELLS_3 24576

/* Rows longer than this many cells (budget_bound + 1) are planned by the long-window kernel:
 * one cooperative grid of CTAs per window (one per SM), each CTA owning a contiguous budget
 * segment in shared memory, with neighbour halos exchanged through an L2 ring (SURVEY.md §8(a)
 * c4). A window whose largest option cost exceeds TURBO_BIG_MAX_COST cells (the halo capacity)
 * is planned instead with its two rows in global memory (L2-resident) and one grid barrier per
 * frame -- same results, slower; no cost is rejected for its size (reading R17). */
#define TURBO_BIG_CELLS 24576
#define TURBO_BIG_MAX_COST 4096
/* Long rows up to this many cells are planned by a thread-block CLUSTER per window instead (up to
 * 16 CTAs, each owning a power-of-two segment of the row in shared memory; the top cells of a
 * segment are pushed into the next CTA's halo through distributed shared memory, costs beyond the
 * halo read the lower segments directly; one split cluster barrier per frame; any option cost):
 * many such windows run at once. Longer rows (e.g. 2^20 cells) keep the grid kernel. Same results
 * either way. */
#define TURBO_CLUSTER_CELLS 131072

/* Number of int64 words of the status vector written by lookup / plan. */
#define TURBO_STATUS_WORDS 2
/* status[0]: smallest frame index whose class id is >= C of its profile (-1 = none);
 *            that frame's option row is written as zeros.
 * status[1]: smallest window index rejected by the planner (negative cost, gain range
 *            rule violated, budget above budget_bound; -1 = none); a rejected window
 *            is planned as all-zero exits, best_gain = best_cost = 0, feasible = 0.
 * The caller initialises both words to -1 (all bits set). */

/* Layout of the statistics vector (a6), int64[TURBO_STATS_WORDS]. */
#define TURBO_STATS_WORDS 181
/* [0,16) exit histogram; [16,176) class x exit histogram for classes 0..9
 * (row-major, 16 exits per class; classes >= 10 not binned); 176 sum best_gain;
 * 177 sum best_cost; 178 #windows; 179 #frames; 180 #infeasible windows. */

/* ---------------------------------------------------------------------------
 * Host-only sizing (no device access). Not a step of the method: it lays out the buffers the
 * steps of PAPER.md:519-525 (§5.2) need -- option blocks, bit-packed choice planes, the long-window
 * scratch -- and the launch shape (row-size classes, serving order). Validates the host copies of
 * profiles and windows, fills windows_host[w].first_option / choice_offset / num_exits /
 * budget_bound / order, and fills *shape (including workspace_bytes).
 * profiles_host: host array of num_profiles descriptors (gain/cost pointers are
 *   not dereferenced here). windows_host: host array, modified in place.
 * Errors: INVALID_ARG (null, K or C out of range, profile index out of range,
 *   num_frames < 0, budget < 0), RANGE (num_frames > 65535, budget >= 2^30). */
turbo_status_t turbo_mckp_workspace(const turbo_profile_t *profiles_host, int32_t num_profiles,
                                    turbo_window_t *windows_host, int32_t num_windows,
                                    turbo_shape_t *shape /* host, out */);

/* ---------------------------------------------------------------------------
 * a1 + a2. a1 (§3; reading R3): if capacity != NULL,
 *   windows[w].budget = max(0, capacity[w] - num_frames_w * base_cost)  (written on device).
 * a2: opt_gain[first_option_w + i*K + k] = gain[class][k],
 *   opt_cost[...] = cost[class][k], class = class_id[first_frame_w + i].
 * profiles: DEVICE array of shape->num_profiles descriptors (same content as the
 * host copy given to turbo_mckp_workspace). windows: device copy of the sized
 * windows. class_id: u8 [total_frames]. opt_gain/opt_cost: int32 [total_options].
 * status: int64[2], see TURBO_STATUS_WORDS. */
turbo_status_t turbo_profile_lookup(const turbo_shape_t *shape /* host */,
                                    const turbo_profile_t *profiles, turbo_window_t *windows,
                                    const uint8_t *class_id, const int32_t *capacity /* nullable */,
                                    int32_t base_cost, int32_t *opt_gain, int32_t *opt_cost,
                                    int64_t *status, turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * a3 + a4 (§5.2 max / s.t., solved exactly = the paper's "upper", PAPER.md:858
 * §6.4; reading R1 f = sum; tie-break R7 / SPEC.md:275): for every window, the suffix max-plus DP
 * over frames N-1..0,
 *   S_N[b] = 0,  S_i[b] = max_{k : c_ik <= b} g_ik + S_{i+1}[b - c_ik]   (b = 0..B),
 * with the per-cell smallest maximising k written bit-packed to the workspace
 * (2 bits for K <= 4, 4 bits otherwise); then G* = S_0[B],
 * C* = min{b : S_0[b] = G*}, feasible = (G* > -inf). Infeasible windows report
 * best_gain = sum_i g_i0, best_cost = sum_i c_i0 (reading R8).
 * workspace: >= shape->workspace_bytes device bytes (choice planes).
 * best_gain, best_cost: int32 [W]; feasible: u8 [W]; status: int64[2]. */
turbo_status_t turbo_mckp_plan(const turbo_shape_t *shape /* host */, const turbo_window_t *windows,
                               const int32_t *opt_gain, const int32_t *opt_cost,
                               void *workspace, size_t workspace_bytes,
                               int32_t *best_gain, int32_t *best_cost, uint8_t *feasible,
                               int64_t *status, turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * a5 ("execute each frame according to the plan": the plan kappa_x of every frame;
 * forward walk = the lexicographic tie-break R7): plan reconstruction from the choice planes of
 * turbo_mckp_plan:
 *   b = C*; for i = 0..N-1: k_i = choice_i[b]; exit_out[first_frame + i] = k_i; b -= c_{i,k_i}.
 * Infeasible or rejected windows get all-zero exits. exit_out: u8 [total_frames]. */
turbo_status_t turbo_backtrack(const turbo_shape_t *shape /* host */, const turbo_window_t *windows,
                               const int32_t *opt_cost, const void *workspace, size_t workspace_bytes,
                               const int32_t *best_cost, const uint8_t *feasible,
                               uint8_t *exit_out, turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * a3 + a4 + a5 fused in one launch (choice planes kept in shared memory when they
 * fit, else in the workspace). Outputs bit-identical to plan + backtrack.
 * workspace may be NULL when shape-dependent turbo_mckp_solve_workspace() returns 0. */
turbo_status_t turbo_mckp_solve(const turbo_shape_t *shape /* host */, const turbo_window_t *windows,
                                const int32_t *opt_gain, const int32_t *opt_cost,
                                void *workspace, size_t workspace_bytes,
                                int32_t *best_gain, int32_t *best_cost, uint8_t *feasible,
                                uint8_t *exit_out, int64_t *status, turbo_stream_t stream);

/* Bytes of workspace turbo_mckp_solve needs for this shape (0 when every window's
 * choice plane fits in shared memory). Host only. */
turbo_status_t turbo_mckp_solve_workspace(const turbo_shape_t *shape, size_t *bytes /* host, out */);

/* Host only (measurement): bytes of choice planes one call writes to HBM -- turbo_mckp_plan
 * (fused = 0: every window) or turbo_mckp_solve / turbo_schedule (fused = 1: the windows whose
 * planes do not stay in shared memory, and every long window). windows_host: the sized host
 * array of turbo_mckp_workspace. The denominator of the choice-plane HBM stream's roofline. */
turbo_status_t turbo_mckp_plane_bytes(const turbo_shape_t *shape, const turbo_window_t *windows_host,
                                      int32_t fused, int64_t *hbm_bytes /* host, out */);

/* ---------------------------------------------------------------------------
 * The whole path a1..a6 in ONE launch (one CTA per window): a1 budget from capacity (when
 * capacity != NULL, written back to windows[w].budget), a2 option rows read straight from
 * class_id and the profiles into shared memory (no option table in HBM; a class >= C sets
 * status[0] and gives a zero row, exactly as turbo_profile_lookup), a3..a5 as
 * turbo_mckp_solve, a6 ACCUMULATED into stats (int64[181], caller zeroes it).
 * Outputs are bit-identical to lookup -> solve -> stats. Workspace as turbo_mckp_solve
 * (turbo_mckp_solve_workspace() bytes). Windows of every size are served: rows up to
 * TURBO_BIG_CELLS cells by one launch per row-size class, longer rows by the cluster kernel
 * (up to TURBO_CLUSTER_CELLS) or the long-window grid kernel, with a1, a2 and a6 fused into them
 * as well. Returns TURBO_ERR_UNSUPPORTED (before any
 * launch) only when a launch cannot fit the device (a long row too large for the grid's shared
 * memory, about 1.8M cells on 148 SMs). */
turbo_status_t turbo_schedule(const turbo_shape_t *shape /* host */, const turbo_profile_t *profiles,
                              turbo_window_t *windows, const uint8_t *class_id,
                              const int32_t *capacity /* nullable */, int32_t base_cost,
                              void *workspace, size_t workspace_bytes,
                              int32_t *best_gain, int32_t *best_cost, uint8_t *feasible,
                              uint8_t *exit_out, int64_t *stats, int64_t *status, turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-3 fused: turbo_schedule taking the discriminator's difficulty scores theta'_x (PAPER.md:525
 * "theta'_x from D_f") instead of class ids. Every kernel that reads a frame's class derives it
 * from its score exactly as turbo_bucketize does (PAPER.md:511 buckets of width bucket_width on
 * d = 1 - theta, reading R6; IEEE float32 decision, NaN -> 0), clamped to the window's profile's
 * C classes, and the DP launch writes the classes to class_out (u8 [total_frames], caller-owned;
 * the walk / statistics kernels read them there). theta: float32 [total_frames]. Outputs are
 * bit-identical to turbo_bucketize -> turbo_schedule with num_classes = C. Other arguments,
 * launches and errors as turbo_schedule. */
turbo_status_t turbo_schedule_theta(const turbo_shape_t *shape /* host */, const turbo_profile_t *profiles,
                                    turbo_window_t *windows, const float *theta, float bucket_width,
                                    uint8_t *class_out, const int32_t *capacity /* nullable */, int32_t base_cost,
                                    void *workspace, size_t workspace_bytes, int32_t *best_gain,
                                    int32_t *best_cost, uint8_t *feasible, uint8_t *exit_out, int64_t *stats,
                                    int64_t *status, turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-1 (comparison arm): the paper's own scheduler, prune-and-search (PAPER.md:539-545,
 * §5.2), on the option tables of turbo_profile_lookup: all frames start at level K-1; while the
 * cost sum_i c_{i,k_i} exceeds the budget, the frame with the minimal marginal gain
 * g_{i,k} - g_{i,k-1} is downgraded one level (ties: larger latency reduction, then smaller frame
 * id); stops when the plan fits or every frame is at level 0 (feasible = 0, plan kept).
 * gain_out/cost_out: int32 [W] (the heuristic plan's totals); feasible: u8 [W];
 * exit_out: u8 [total_frames]; steps: int32 [W] downgrade steps (nullable).
 * Shared memory holds one byte per frame per warp: UNSUPPORTED if max_frames is too large. */
turbo_status_t turbo_heuristic_plan(const turbo_shape_t *shape /* host */, const turbo_window_t *windows,
                                    const int32_t *opt_gain, const int32_t *opt_cost, int32_t *gain_out,
                                    int32_t *cost_out, uint8_t *feasible, uint8_t *exit_out,
                                    int32_t *steps /* nullable */, turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-3 (the step before the path): difficulty score -> difficulty class. PAPER.md:511
 * buckets of width 0.1; theta'_x from D_f (:525); reading R6: class = bucket of d = 1 - theta,
 * class_out[x] = clamp(floor((1 - theta[x]) * (1 / bucket_width)), 0, C-1), decided in IEEE
 * float32 (1/bucket_width rounded to float32 once); NaN -> 0. theta: float32 [n], 16-B aligned;
 * class_out: u8 [n], 4-B aligned. */
turbo_status_t turbo_bucketize(const float *theta, int64_t num_frames, int32_t num_classes,
                               float bucket_width, uint8_t *class_out, turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * NEXT-2 (the step after the path): plan -> per-exit batches ("organize the frames
 * assigned by the same enhancement level to execute in a batch", :545). Per window w:
 * count_out[16 w + k] = n_k, the number of frames planned at level k; order_out[first_frame_w
 * + j] = window-local frame indices grouped by level ascending, arrival order inside a level
 * (a stable partition; the batch of level k starts at sum_{k' < k} n_k'). exit_out: the plan
 * (u8 [total_frames]); count_out: int32 [16 W]; order_out: int32 [total_frames].
 * Executed latency (optional, latency_out != NULL): latency_out[w] = f = sum_{k < K_w} I_k(n_k),
 * the GPU time of running the window's batches (PAPER.md:525 f(.) of the constraint), with I_k(n)
 * from batch_cost in the layout of turbo_batched_plan (profile p at p * 16 * (batch_cap + 1),
 * row k = I_k(0 .. batch_cap)); int64 [W]. A window with some n_k > batch_cap gets latency -1 and
 * sets status[1] (min window index; int64[2], required with latency_out). With linear tables
 * (I_k(n) = n c_k) f is the plan's summed per-frame cost (reading R1). */
turbo_status_t turbo_batches(const turbo_shape_t *shape /* host */, const turbo_window_t *windows,
                             const uint8_t *exit_out, int32_t *count_out, int32_t *order_out,
                             const int32_t *batch_cost /* nullable */, int32_t batch_cap,
                             int64_t *latency_out /* nullable */, int64_t *status /* nullable */,
                             turbo_stream_t stream);

/* ---------------------------------------------------------------------------
 * a6 (per GPU): ACCUMULATES the plan statistics into stats (int64[181], layout
 * above; caller zeroes it): the per-exit usage and per-difficulty-class x exit histograms and
 * the totals the paper's scheduler evaluation reports per run (accuracy gain, GPU time of the
 * chosen enhancement, infeasible windows; PAPER.md:561-562 §6, :858 §6.4). Not part of the
 * optimisation itself. The cross-GPU sum (one allreduce over NVLink) is done by
 * the caller's communicator, not inside the library. */
turbo_status_t turbo_stats(const turbo_shape_t *shape /* host */, const turbo_window_t *windows,
                           const uint8_t *class_id, const uint8_t *exit_out,
                           const int32_t *best_gain, const int32_t *best_cost,
                           const uint8_t *feasible, int64_t *stats, turbo_stream_t stream);

/* NEXT-4: exact plans under the paper's batched latency constraint:
 * cost(plan) = sum_k I_k(n_k), n_k = frames planned at level k, I_k(n) = the latency of a batch of
 * n frames at level k (latency independent of content :103). Result per window:
 * larger gain, then smaller cost, then the count vector (n_{K-1}, ..., n_0) lexicographically
 * smaller, then the assignment: frames in canonical order (class, then arrival index) x_0 ..
 * x_{N-1}; backwards from x_{N-1}, each takes the highest level that keeps the plan optimal
 * (reading R20). When the gains have increasing differences in the class,
 * g[c+1][k+1] - g[c+1][k] >= g[c][k+1] - g[c][k] (R19), this is the canonical
 * assignment (sorted frames fill level 0, then 1, ...; R18) and the count vectors are enumerated
 * directly; windows WITHOUT R19 are solved by the program over the canonical prefix and its count
 * vector (every transportation optimum at once), which needs `workspace` (device, >=
 * turbo_batched_workspace() bytes; K <= 8, C <= 16). Without a workspace such windows are rejected.
 * Preconditions: |g| <= 2^24, sum over the window's frames of |g| per level <= 2^30, batch
 * latencies in [0, 2^26]; a window violating them (or with budget < 0) is planned all-zero,
 * feasible = 0, gain = cost = 0, and status[1] = min such window; a class id >= C sets status[0]
 * like the lookup. batch_cost (device int32): per profile p a table at p * 16 * (batch_cap + 1),
 * row k (k < K_p) = I_k(0 .. batch_cap). Host checks (TURBO_ERR_UNSUPPORTED): max_frames <=
 * batch_cap <= 255, C(max_frames + max_exits - 1, max_exits - 1) <= 2^26 count vectors per window
 * and (max_frames + 1)^(max_exits - 1) < 2^62. Infeasible windows: all frames at level 0,
 * feasible = 0, best_gain = sum g[c_x][0], best_cost = I_0(N). Budgets are read from
 * windows[w].budget (set them on the device, or a1 via turbo_profile_lookup). Stream-ordered. */
turbo_status_t turbo_batched_plan(const turbo_shape_t *shape /* host */, const turbo_window_t *windows,
                                  const turbo_profile_t *profiles /* device */, const int32_t *batch_cost,
                                  int32_t batch_cap, const uint8_t *class_id, void *workspace /* nullable */,
                                  size_t workspace_bytes, int32_t *best_gain, int32_t *best_cost,
                                  uint8_t *feasible, uint8_t *exit_out, int64_t *status, turbo_stream_t stream);

/* Bytes of device workspace turbo_batched_plan needs to plan windows without R19 for this shape
 * (0: the shape is too large for that program -- such windows are then rejected). Host only. */
turbo_status_t turbo_batched_workspace(const turbo_shape_t *shape, size_t *bytes /* host, out */);

/* Copy `bytes` from src to dst with the SMs (one kernel on `stream`) instead of a copy engine.
 * Both pointers must be device-accessible: device memory, or pinned host memory (cudaHostAlloc /
 * torch pin_memory, mapped through unified addressing). Not a step of the method: the transfer of
 * a serving loop's per-step inputs and results, a few tens of KB, where a copy-engine transfer's
 * fixed latency dominates. INVALID_ARG for NULL pointers with bytes > 0. */
turbo_status_t turbo_memcpy_sm(void *dst, const void *src, size_t bytes, turbo_stream_t stream);

/* Debug / test hook: force a DP kernel variant. variant & 3: 0 = automatic, 1 = fused solve
 * keeps choice planes in shared memory (when they fit the per-CTA maximum), 2 = in HBM;
 * variant & 4: do not stage option tables in shared memory (shuffle broadcast instead);
 * variant & 8: use the lockstep multi-window kernel (dp_pack.cu; V windows per CTA) for
 * single-class short-row batches instead of one CTA per window;
 * variant & 16: the runtime-K kernel also for row class 3 of mixed-K plan launches;
 * variant & 32: never the runtime-K body (the fifteen K-specific bodies everywhere);
 * variant & 64: turbo_batched_plan plans every valid window with the general program (R20);
 * variant & 128: u16 rows (NEXT-5) for the windows that qualify in the fixed-K CTA kernels with
 *   staged options and the walk in the kernel -- gains >= 0, a cost-0 exit in every frame,
 *   sum_i max_k g + max g + 1 <= 65535. Opt-in: measured slower than the int32 rows on c2 (the
 *   two-cells-per-word unpack costs more instructions than the halved shared loads save);
 * variant & 256: never the 72-register kernels (fixed-K fused solve and runtime-K) for launches of
 *   <= 4 warps per window;
 * variant & 512: long rows all on the grid kernel (no cluster kernel).
 * Returns INVALID_ARG for other values. Process-wide; not needed in production. */
turbo_status_t turbo_debug_set_variant(int32_t variant);

/* Debug / profiling hook: with trace != NULL (device memory, `words` int64 entries, caller-owned,
 * zeroed by the caller) the CTA DP kernels record, for window w, %globaltimer nanoseconds at
 * trace[8w + p]: p = 0 window start, 1 prologue done, 2 DP done, 3 optimum done, 4 plan
 * reconstructed (fused kernels), 5 window end. NULL disables (the default). Process-wide; not
 * needed in production. Returns TURBO_ERR_UNSUPPORTED unless the library was built with
 * TURBO_TRACE defined (the marks are compiled out of production builds). */
turbo_status_t turbo_debug_trace(int64_t *trace, int64_t words);
/* Test hook: with counter != NULL (device memory, one int64, caller-owned and zeroed) every DP
 * kernel launch that follows adds 1 per window it planned on u16 rows (NEXT-5, opt-in with
 * turbo_debug_set_variant bit 128), so tests can prove which row format served a batch. NULL
 * disables (the default). Process-wide; not needed in production. */
turbo_status_t turbo_debug_u16_counter(int64_t *counter);
/* Measurement hook (not a step of the method): the shared-memory roofline denominator. Launches
 * ctas_per_sm (1 or 2) x SMs CTAs of 1024 threads, each thread issuing iters x 32 conflict-free
 * shared loads of bytes_per_lane (4, 8 or 16) bytes (4: one 128-B wavefront per warp instruction,
 * the DP's access type); *bytes_out (host) = bytes the launch reads. The caller times the launch
 * (CUDA events) and divides. sink: device, >= 4 KB, never meaningfully written. */
turbo_status_t turbo_debug_smem_stream(int32_t iters, int32_t ctas_per_sm, int32_t bytes_per_lane, void *sink,
                                       double *bytes_out, turbo_stream_t stream);
/* Test hook: launches one kernel whose bounds check is violated on purpose. In the checked build
 * (TURBO_CHECKS) it prints one "TCHECK" report; in the production build it does nothing. */
turbo_status_t turbo_debug_tcheck_selftest(turbo_stream_t stream);
/* Kernels this library has launched so far in the process (all threads and devices; graph
 * capture counts the captured launches once). Lets a caller count the kernels of a call. */
int64_t turbo_launch_count(void);
const char *turbo_status_string(turbo_status_t s);
int32_t turbo_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TURBO_H */

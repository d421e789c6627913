// api.cu -- host side of the C ABI (include/turbo.h): validation, sizing, dispatch.
// No device memory is allocated here and nothing synchronises the device.
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <algorithm>
#include <climits>
#include <atomic>

#include "turbo_internal.cuh"

namespace turbo {

struct DeviceInfo {
    int num_sms = 0;
    int smem_per_sm = 0;
    int smem_per_cta_optin = 0;
};

static std::mutex g_mu;
static DeviceInfo g_dev[64];
static int g_variant = 0;

static cudaError_t device_info(DeviceInfo *out)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_dev[dev].num_sms == 0) {
        DeviceInfo d;
        if ((e = cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&d.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev)) !=
            cudaSuccess)
            return e;
        if ((e = cudaDeviceGetAttribute(&d.smem_per_cta_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) !=
            cudaSuccess)
            return e;
        g_dev[dev] = d;
    }
    *out = g_dev[dev];
    return cudaSuccess;
}

// smem words per CTA for the DP: row, option table (osm) or backtrack costs, choice planes
static const int64_t OSM_LIMIT_BYTES = 48 * 1024;   // largest per-window option table staged in smem

static void dp_smem_words(const turbo_shape_t *s, int mode, DpParams *P)
{
    const int64_t rows = (num_rows(s->max_budget_small) + 15) & ~(int64_t)15;   // whole tiles (<= 16 rows)
    P->row_words = (int32_t)(rows * 32);
    const int rpt_min = s->max_exits <= 4 ? 16 : 8;
    const int64_t tiles = (rows + rpt_min - 1) / rpt_min;
    const int64_t chs = mode == DP_SOLVE_SMEM ? (int64_t)s->max_frames * tiles * 32 : 0;
    P->chs_words = (int32_t)(chs > INT32_MAX ? INT32_MAX : chs);
    const int64_t opts = s->max_options;
    // stage the option table only when it is small next to the row(s) it feeds: for short rows
    // the table would dominate shared memory and cap residency; those windows broadcast options
    // from registers (shuffles) instead
    const int64_t row_bytes = (int64_t)P->row_words * 4 * (dp_warps_per_window(s) > 1 ? 2 : 1);
    P->osm = (opts * 8 <= OSM_LIMIT_BYTES && opts * 8 <= (row_bytes > 4096 ? row_bytes : 4096) &&
              !(g_variant & 4)) ? 1 : 0;
    P->cst_words = P->osm ? (int32_t)(2 * opts) : 0;   // words after the rows: the staged option table
    P->max_options = (int32_t)opts;
}

// -inf pad below each row: shifts up to this many cells need no bounds check (one 4-bit tile;
// capped by the row itself, since a shift above B + 1 is never feasible anyway)
static int32_t dp_pad_words(const turbo_shape_t *s)
{
    const int64_t row = num_rows(s->max_budget_small) * 32;
    return (int32_t)(row < 256 ? row : 256);
}

// Per-device streams and events used to run the row-size class launches concurrently.
struct ForkJoin {
    cudaStream_t streams[TURBO_NUM_CLASSES];
    cudaEvent_t fork;
    cudaEvent_t join[TURBO_NUM_CLASSES];
};

// Per calling THREAD and device: concurrent callers (or one thread capturing a graph while another
// launches eagerly) never share a library stream. The streams live as long as the process.
static ForkJoin *fork_join_for_device()
{
    thread_local ForkJoin *per_dev[64] = {nullptr};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!per_dev[dev]) {
        ForkJoin *fj = new ForkJoin();
        for (int c = 0; c < TURBO_NUM_CLASSES; ++c) {
            if (cudaStreamCreateWithFlags(&fj->streams[c], cudaStreamNonBlocking) != cudaSuccess) return nullptr;
            if (cudaEventCreateWithFlags(&fj->join[c], cudaEventDisableTiming) != cudaSuccess) return nullptr;
        }
        if (cudaEventCreateWithFlags(&fj->fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        per_dev[dev] = fj;
    }
    return per_dev[dev];
}

// fused solve keeps choice planes in shared memory when they are at most this many bytes or
// twice the row(s): otherwise they would cap the CTAs resident per SM (and HBM/L2 is fine)
static int64_t smem_choice_floor = 16 * 1024;

static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace turbo

using namespace turbo;

extern "C" {

int32_t turbo_abi_version(void) { return 1; }

const char *turbo_status_string(turbo_status_t s)
{
    switch (s) {
        case TURBO_OK: return "ok";
        case TURBO_ERR_INVALID_ARG: return "invalid argument";
        case TURBO_ERR_RANGE: return "value out of range";
        case TURBO_ERR_WORKSPACE: return "workspace too small";
        case TURBO_ERR_CUDA: return "CUDA error";
        case TURBO_ERR_UNSUPPORTED: return "unsupported shape";
    }
    return "unknown";
}

int64_t turbo_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

static int64_t *g_trace = nullptr;
static int64_t g_trace_words = 0;

turbo_status_t turbo_debug_trace(int64_t *trace, int64_t words)
{
#ifndef TURBO_TRACE
    if (trace != nullptr) return TURBO_ERR_UNSUPPORTED;   // library built without the marks
#endif
    if (trace != nullptr && words < 8) return TURBO_ERR_INVALID_ARG;
    g_trace = trace;
    g_trace_words = trace ? words : 0;
    return TURBO_OK;
}

static int64_t *g_u16_count = nullptr;

turbo_status_t turbo_debug_u16_counter(int64_t *counter)
{
    g_u16_count = counter;
    return TURBO_OK;
}

turbo_status_t turbo_debug_set_variant(int32_t variant)
{
    if (variant < 0 || variant > 1023 || (variant & 3) == 3) return TURBO_ERR_INVALID_ARG;
    g_variant = variant;
    return TURBO_OK;
}

turbo_status_t turbo_mckp_workspace(const turbo_profile_t *profiles_host, int32_t num_profiles,
                                    turbo_window_t *windows_host, int32_t num_windows, turbo_shape_t *shape)
{
    if (!shape || num_profiles < 0 || num_windows < 0) return TURBO_ERR_INVALID_ARG;
    if ((num_profiles > 0 && !profiles_host) || (num_windows > 0 && !windows_host)) return TURBO_ERR_INVALID_ARG;
    for (int32_t p = 0; p < num_profiles; ++p) {
        const turbo_profile_t &pr = profiles_host[p];
        if (pr.num_exits < 2 || pr.num_exits > MAX_EXITS) return TURBO_ERR_INVALID_ARG;
        if (pr.num_classes < 1 || pr.num_classes > 256) return TURBO_ERR_INVALID_ARG;
        if (!pr.gain || !pr.cost) return TURBO_ERR_INVALID_ARG;
    }
    turbo_shape_t s;
    std::memset(&s, 0, sizeof(s));
    s.num_windows = num_windows;
    s.num_profiles = num_profiles;
    s.min_exits = MAX_EXITS;
    s.max_exits = 2;
    for (int c = 0; c < TURBO_NUM_CLASSES; ++c) {
        s.cls_min_exits[c] = MAX_EXITS;
        s.cls_max_exits[c] = 2;
    }
    int64_t opt = 0, ws = 0, frames = 0, cells = 0;
    for (int32_t w = 0; w < num_windows; ++w) {
        turbo_window_t &win = windows_host[w];
        if (win.profile < 0 || win.profile >= num_profiles) return TURBO_ERR_INVALID_ARG;
        if (win.num_frames < 0 || win.budget < 0 || win.first_frame < 0) return TURBO_ERR_INVALID_ARG;
        if (win.num_frames > 65535 || win.budget >= (1 << 30)) return TURBO_ERR_RANGE;
        const int K = profiles_host[win.profile].num_exits;
        win.num_exits = K;
        win.budget_bound = win.budget;
        win.first_option = opt;
        win.choice_offset = ws;
        win.order = w;
        opt += ((int64_t)win.num_frames * K + 3) & ~(int64_t)3;    // 16-B aligned option blocks
        ws += choice_plane_bytes(win.num_frames, win.budget, K);
        frames = frames > win.first_frame + win.num_frames ? frames : win.first_frame + win.num_frames;
        cells += (int64_t)win.num_frames * ((int64_t)win.budget + 1);
        if (win.num_frames > s.max_frames) s.max_frames = win.num_frames;
        if ((int64_t)win.num_frames * K > s.max_options) s.max_options = win.num_frames * K;
        if (win.budget > s.max_budget) s.max_budget = win.budget;
        const int rc = row_class((int64_t)win.budget + 1);
        if (rc >= TURBO_NUM_CLASSES) {
            s.num_big += 1;
        } else {
            if (win.budget > s.max_budget_small) s.max_budget_small = win.budget;
            s.cls_count[rc] += 1;
            if (win.budget > s.cls_max_budget[rc]) s.cls_max_budget[rc] = win.budget;
            if (win.num_frames > s.cls_max_frames[rc]) s.cls_max_frames[rc] = win.num_frames;
            if (win.num_frames * K > s.cls_max_options[rc]) s.cls_max_options[rc] = win.num_frames * K;
            if (K < s.cls_min_exits[rc]) s.cls_min_exits[rc] = K;
            if (K > s.cls_max_exits[rc]) s.cls_max_exits[rc] = K;
        }
        if (K < s.min_exits) s.min_exits = K;
        if (K > s.max_exits) s.max_exits = K;
        if (profiles_host[win.profile].num_classes > s.num_classes_max)
            s.num_classes_max = profiles_host[win.profile].num_classes;
    }
    if (num_windows == 0) s.min_exits = s.max_exits = 2;
    // Serving order (turbo_window_t.order): windows grouped by row-size class (the long ones
    // last), largest work first inside a class -- the CTA scheduler hands out blocks in index
    // order, so the longest windows start first and the short ones fill the gaps (LPT). Used
    // when there are several classes or the work inside a class is uneven.
    {
        std::vector<std::pair<int64_t, int32_t>> key((size_t)num_windows);
        int n_cls = s.num_big > 0 ? 1 : 0;
        for (int c = 0; c < TURBO_NUM_CLASSES; ++c) n_cls += s.cls_count[c] ? 1 : 0;
        bool uneven = false;
        int64_t wmin[TURBO_NUM_CLASSES + 1], wmax[TURBO_NUM_CLASSES + 1];
        for (int c = 0; c <= TURBO_NUM_CLASSES; ++c) {
            wmin[c] = INT64_MAX;
            wmax[c] = 0;
        }
        for (int32_t w = 0; w < num_windows; ++w) {
            const turbo_window_t &win = windows_host[w];
            const int rc = std::min(row_class((int64_t)win.budget_bound + 1), TURBO_NUM_CLASSES);
            const int64_t work = (int64_t)win.num_frames * ((int64_t)win.budget_bound + 1) * (win.num_exits + 1);
            wmin[rc] = std::min(wmin[rc], work);
            wmax[rc] = std::max(wmax[rc], work);
            // class ascending, work descending, index ascending (deterministic)
            key[(size_t)w] = std::make_pair(((int64_t)rc << 58) | ((((int64_t)1 << 58) - 1) - std::min(work, ((int64_t)1 << 58) - 1)), w);
        }
        for (int c = 0; c <= TURBO_NUM_CLASSES; ++c)
            if (wmax[c] > 0 && wmax[c] * 2 > wmin[c] * 3) uneven = true;
        // class launch order: longest rows first, so the short-row classes fill the SMs the
        // longest-row launch leaves idle in its last wave (c5, 16,384 windows, same box: 13.44 vs
        // 13.52 ms smallest-first; scripts/cls_order.py). (Round 1, 2,048 windows: heaviest-window-
        // first by N (B+1) (K+1) ACROSS classes was slower, 2.63 vs 2.53 ms.)
        s.cls_order = 0x0123;
        s.ordered = (n_cls > 1 || uneven) ? 1 : 0;
        if (s.ordered) {
            std::sort(key.begin(), key.end());
            for (int32_t r = 0; r < num_windows; ++r) windows_host[r].order = key[(size_t)r].second;
        }
    }
    s.total_frames = frames;
    s.total_options = opt;
    s.total_cells = cells;
    if (s.num_big > 0) {                 // long-window kernel scratch: flags + halo ring
        s.grid_scratch_offset = (ws + 255) & ~(int64_t)255;
        ws = s.grid_scratch_offset + grid_scratch_bytes(s.max_budget);
    }
    s.workspace_bytes = ws;
    *shape = s;
    return TURBO_OK;
}

turbo_status_t turbo_profile_lookup(const turbo_shape_t *shape, const turbo_profile_t *profiles,
                                    turbo_window_t *windows, const uint8_t *class_id, const int32_t *capacity,
                                    int32_t base_cost, int32_t *opt_gain, int32_t *opt_cost, int64_t *status,
                                    turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!profiles || !windows || !status || base_cost < 0) return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && !class_id) return TURBO_ERR_INVALID_ARG;
    if (shape->total_options > 0 && (!opt_gain || !opt_cost)) return TURBO_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(opt_gain) | reinterpret_cast<uintptr_t>(opt_cost)) & 15)
        return TURBO_ERR_INVALID_ARG;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    cudaError_t e = launch_lookup(profiles, windows, shape->num_windows, class_id, capacity, base_cost, opt_gain,
                                  opt_cost, status, shape->max_options, d.num_sms, (cudaStream_t)stream);
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

// Launch shape of one row-size class: windows outside the class are skipped by the kernel.
static turbo_shape_t class_shape(const turbo_shape_t *s, int c)
{
    turbo_shape_t t = *s;
    t.max_budget_small = s->cls_max_budget[c];
    t.max_budget = s->cls_max_budget[c];
    t.max_frames = s->cls_max_frames[c];
    t.max_options = s->cls_max_options[c];
    t.min_exits = s->cls_min_exits[c];
    t.max_exits = s->cls_max_exits[c];
    t.num_big = 0;
    return t;
}

enum { RUN_PLAN = 0, RUN_SOLVE = 1, RUN_SCHEDULE = 2 };

// Fused-solve variant of one class: choice planes in shared memory when they fit under
// smem_choice_floor bytes or twice the rows (or, forced by the debug hook, up to the per-CTA max).
static int solve_mode(const turbo_shape_t *cs)
{
    if ((g_variant & 3) == 2) return DP_SOLVE_GLOBAL;
    DpParams P;
    std::memset(&P, 0, sizeof(P));
    dp_smem_words(cs, DP_SOLVE_SMEM, &P);
    P.pad_words = dp_pad_words(cs);
    const int64_t bytes = (int64_t)dp_smem_bytes(P, dp_warps_per_window(cs));
    DeviceInfo d;
    // planes in smem only when the whole CTA still fits (2-bit planes of long rows are below
    // twice the rows yet over the per-CTA maximum with them)
    const bool fits = device_info(&d) == cudaSuccess && bytes + 1024 <= (int64_t)d.smem_per_cta_optin;
    if ((g_variant & 3) == 1) return fits ? DP_SOLVE_SMEM : DP_SOLVE_GLOBAL;
    const int64_t planes = (int64_t)P.chs_words * 4;
    const int64_t rows = bytes - planes;
    return fits && (planes <= smem_choice_floor || planes <= 2 * rows) ? DP_SOLVE_SMEM : DP_SOLVE_GLOBAL;
}

// Does a fused solve / schedule of this batch write any choice plane to HBM?
static bool solve_needs_workspace(const turbo_shape_t *s)
{
    if (s->num_big > 0) return true;
    for (int c = 0; c < TURBO_NUM_CLASSES; ++c) {
        if (!s->cls_count[c]) continue;
        const turbo_shape_t cs = class_shape(s, c);
        if (solve_mode(&cs) == DP_SOLVE_GLOBAL) return true;
    }
    return false;
}

// One launch per non-empty row-size class (then the grid kernel for long windows).
static turbo_status_t run_dp(const turbo_shape_t *shape, int kind, const DpParams &base, turbo_stream_t stream)
{
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    // long windows (the grid kernel) are validated first: nothing is launched unless every launch
    // of the call can run
    const int grid_mode = kind == RUN_PLAN ? DP_PLAN : DP_SOLVE_GLOBAL;
    if (shape->num_big > 0) {
        const cudaError_t ge = check_dp_grid(shape, grid_mode, d.num_sms, d.smem_per_cta_optin, base.cluster_cap);
        if (ge != cudaSuccess) {
            cudaGetLastError();
            return ge == cudaErrorInvalidConfiguration || ge == cudaErrorCooperativeLaunchTooLarge
                       ? TURBO_ERR_UNSUPPORTED : TURBO_ERR_CUDA;
        }
    }
    DpParams Ps[TURBO_NUM_CLASSES];
    turbo_shape_t shapes[TURBO_NUM_CLASSES];
    int modes[TURBO_NUM_CLASSES];
    bool walk[TURBO_NUM_CLASSES];
    for (int c = 0; c < TURBO_NUM_CLASSES; ++c) {          // validate every class before launching
        walk[c] = false;
        if (!shape->cls_count[c]) continue;
        shapes[c] = class_shape(shape, c);
        modes[c] = kind == RUN_PLAN ? DP_PLAN : solve_mode(&shapes[c]);
        // choice planes in HBM: the DP runs in plan mode and a separate kernel walks the planes
        // (thousands of latency-bound walks in flight instead of one per DP CTA slot)
        if (modes[c] == DP_SOLVE_GLOBAL) {
            modes[c] = DP_PLAN;
            walk[c] = true;
        }
        DpParams &P = Ps[c];
        P = base;
        dp_smem_words(&shapes[c], modes[c], &P);
        P.warp_words = 0;
        P.pad_words = dp_pad_words(&shapes[c]);
        if (kind == RUN_SCHEDULE && P.osm) {
            // fused scratch after the option table: profile (C*K int2), class ids and exits (N B each)
            P.prof_entries = shapes[c].num_classes_max * shapes[c].max_exits;
            P.cst_words += 2 * P.prof_entries + 2 * ((shapes[c].max_frames + 3) / 4);
        }
        P.cls = c;
        P.max_frames = shapes[c].max_frames;
        // mixed-K plan-mode launches of row classes 0-2 run the runtime-K kernel: several CTAs of
        // different K per SM would thrash the instruction cache with fifteen unrolled bodies, and
        // 128 registers per thread would cap their residency (c5, ncu: class 0 2.42 -> 0.61 ms,
        // class 1 2.56 -> 1.06, class 2 4.02 -> 3.28). The longest rows (one CTA per SM, so one K
        // per SM) keep the K-specific bodies (runtime-K measured 11.2 vs 8.4 ms there).
        P.generic = (modes[c] == DP_PLAN && !dp_kernel_fixed_k(shapes[c].min_exits, shapes[c].max_exits) &&
                     (c < 3 || (g_variant & 16)) && !(g_variant & 32)) ? 1 : 0;
        P.cls_count = shape->cls_count[c];
        // the serving order is followed by the mixed-K kernels; fixed-K kernels go in index order
        P.ordered = (shape->ordered && !dp_kernel_fixed_k(shapes[c].min_exits, shapes[c].max_exits)) ? 1 : 0;
        P.cls_first = 0;
        for (int c2 = 0; c2 < c; ++c2) P.cls_first += shape->cls_count[c2];
        const cudaError_t ce = check_dp(&shapes[c], modes[c], P, d.smem_per_cta_optin);   // incl. static smem
        if (ce == cudaErrorInvalidConfiguration) return TURBO_ERR_UNSUPPORTED;
        if (ce != cudaSuccess) return TURBO_ERR_CUDA;
    }
    DpLaunch info;
    cudaError_t e = cudaSuccess;
    auto launch_walk = [&](int c, cudaStream_t st) -> cudaError_t {
        if (!walk[c]) return cudaSuccess;
        const DpParams &P = Ps[c];
        WinSel sel;
        sel.cls = c;
        sel.ordered = P.ordered;
        sel.first = P.cls_first;
        sel.count = P.cls_count;
        if (kind == RUN_SCHEDULE)
            return launch_walk_sched(P.windows, shape->num_windows, P.profiles, P.class_id, P.workspace, P.best_gain,
                                     P.best_cost, P.feasible, P.exit_out, P.stats, d.num_sms, st, sel);
        return launch_backtrack(P.windows, shape->num_windows, P.opt_cost, P.workspace, P.best_cost, P.feasible,
                                P.exit_out, d.num_sms, st, sel);
    };
    int n_cls = 0;
    for (int c = 0; c < TURBO_NUM_CLASSES; ++c) n_cls += shape->cls_count[c] ? 1 : 0;
    if (n_cls <= 1) {
        for (int c = 0; c < TURBO_NUM_CLASSES && e == cudaSuccess; ++c)
            if (shape->cls_count[c]) {
                // opt-in (variant & 8): the lockstep kernel (V windows per CTA, one barrier per frame
                // for all of them). Measured slower on c2 (42.7 vs 37.2 us): the shared
                // per-frame barrier drains and refills the whole SM's shared-memory pipe every frame
                int pv, pt, pw;
                size_t ps;
                if (modes[c] == DP_SOLVE_SMEM && shape->num_big == 0 && (g_variant & 8) &&
                    pack_geometry(&shapes[c], Ps[c], d.num_sms, d.smem_per_cta_optin, &pv, &pt, &pw, &ps)) {
                    e = launch_pack(&shapes[c], Ps[c], d.num_sms, d.smem_per_cta_optin, (cudaStream_t)stream);
                    continue;
                }
                e = launch_dp(&shapes[c], modes[c], Ps[c], d.num_sms, d.smem_per_sm, d.smem_per_cta_optin,
                              (cudaStream_t)stream, &info);
                if (e == cudaSuccess) e = launch_walk(c, (cudaStream_t)stream);
            }
    } else {
        // Several classes: each class launch is bounded by its longest window's frame chain, so the
        // launches run CONCURRENTLY on library-owned streams forked from (and joined back into) the
        // caller's stream with events -- stream-ordered for the caller and capturable in graphs.
        ForkJoin *fj = fork_join_for_device();
        if (!fj) return TURBO_ERR_CUDA;
        e = cudaEventRecord(fj->fork, (cudaStream_t)stream);
        int order = shape->cls_order, seen = 0;                     // a permutation, else 0 1 2 3
        for (int i = 0; i < TURBO_NUM_CLASSES; ++i) seen |= 1 << ((order >> (4 * i)) & 15);
        if (seen != (1 << TURBO_NUM_CLASSES) - 1) order = 0x3210;
        for (int i = 0; i < TURBO_NUM_CLASSES && e == cudaSuccess; ++i) {
            const int c = (order >> (4 * i)) & 15;
            if (c >= TURBO_NUM_CLASSES || !shape->cls_count[c]) continue;
            if ((e = cudaStreamWaitEvent(fj->streams[c], fj->fork, 0)) != cudaSuccess) break;
            // every forked stream is joined back below, also when a launch on it fails (an unjoined
            // stream would break the caller's graph capture)
            e = launch_dp(&shapes[c], modes[c], Ps[c], d.num_sms, d.smem_per_sm, d.smem_per_cta_optin,
                          fj->streams[c], &info);
            if (e == cudaSuccess) e = launch_walk(c, fj->streams[c]);
            cudaError_t je = cudaEventRecord(fj->join[c], fj->streams[c]);
            if (je == cudaSuccess) je = cudaStreamWaitEvent((cudaStream_t)stream, fj->join[c], 0);
            if (e == cudaSuccess) e = je;
        }
    }
    if (e == cudaSuccess && shape->num_big > 0) {          // long windows: the whole grid per window
        DpParams P = base;
        P.grid_scratch_offset = shape->grid_scratch_offset;
        e = launch_dp_grid(shape, grid_mode, P, d.num_sms, d.smem_per_cta_optin, (cudaStream_t)stream);
    }
    if (e == cudaErrorInvalidConfiguration || e == cudaErrorCooperativeLaunchTooLarge) {
        cudaGetLastError();
        return TURBO_ERR_UNSUPPORTED;
    }
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

static DpParams base_params(const turbo_shape_t *shape, const turbo_window_t *windows, const int32_t *opt_gain,
                            const int32_t *opt_cost, void *workspace, int32_t *best_gain, int32_t *best_cost,
                            uint8_t *feasible, uint8_t *exit_out, int64_t *status)
{
    DpParams P;
    std::memset(&P, 0, sizeof(P));
    P.windows = windows;
    P.num_windows = shape->num_windows;
    P.opt_gain = opt_gain;
    P.opt_cost = opt_cost;
    P.workspace = reinterpret_cast<uint8_t *>(workspace);
    P.best_gain = best_gain;
    P.best_cost = best_cost;
    P.feasible = feasible;
    P.exit_out = exit_out;
    P.status = status;
    P.grid_scratch_offset = shape->grid_scratch_offset;
    P.cls = -1;
    static int dbg = -1;                     // TURBO_DP_DEBUG: timing-only switches (8: no stats
    if (dbg < 0) {                           // flush, 16: no backtrack); results are then wrong
        const char *e = getenv("TURBO_DP_DEBUG");
        dbg = e ? atoi(e) : 0;
    }
    P.debug = dbg;
    P.u16 = (g_variant & 128) ? 1 : 0;                 // NEXT-5 u16 rows: opt-in
    P.u16_count = g_u16_count;
    P.small = (g_variant & 256) ? 0 : 1;
    P.cluster_cap = (g_variant & 512) ? 0 : TURBO_CLUSTER_CELLS;   // variant 512: the grid kernel only
    P.trace = g_trace;
    P.trace_words = g_trace_words;
    return P;
}

turbo_status_t turbo_mckp_plan(const turbo_shape_t *shape, const turbo_window_t *windows, const int32_t *opt_gain,
                               const int32_t *opt_cost, void *workspace, size_t workspace_bytes,
                               int32_t *best_gain, int32_t *best_cost, uint8_t *feasible, int64_t *status,
                               turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!windows || !best_gain || !best_cost || !feasible || !status) return TURBO_ERR_INVALID_ARG;
    if (shape->total_options > 0 && (!opt_gain || !opt_cost)) return TURBO_ERR_INVALID_ARG;
    if ((int64_t)workspace_bytes < shape->workspace_bytes || (shape->workspace_bytes > 0 && !workspace))
        return TURBO_ERR_WORKSPACE;
    return run_dp(shape, RUN_PLAN,
                  base_params(shape, windows, opt_gain, opt_cost, workspace, best_gain, best_cost, feasible, nullptr,
                              status),
                  stream);
}

turbo_status_t turbo_backtrack(const turbo_shape_t *shape, const turbo_window_t *windows, const int32_t *opt_cost,
                               const void *workspace, size_t workspace_bytes, const int32_t *best_cost,
                               const uint8_t *feasible, uint8_t *exit_out, turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!windows || !best_cost || !feasible) return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && !exit_out) return TURBO_ERR_INVALID_ARG;
    if (shape->total_options > 0 && !opt_cost) return TURBO_ERR_INVALID_ARG;
    if ((int64_t)workspace_bytes < shape->workspace_bytes || (shape->workspace_bytes > 0 && !workspace))
        return TURBO_ERR_WORKSPACE;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    cudaError_t e = launch_backtrack(windows, shape->num_windows, opt_cost,
                                     reinterpret_cast<const uint8_t *>(workspace), best_cost, feasible, exit_out,
                                     d.num_sms, (cudaStream_t)stream);
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

turbo_status_t turbo_mckp_plane_bytes(const turbo_shape_t *shape, const turbo_window_t *windows_host,
                                      int32_t fused, int64_t *hbm_bytes)
{
    if (!shape || !hbm_bytes || (shape->num_windows > 0 && !windows_host)) return TURBO_ERR_INVALID_ARG;
    bool hbm_class[TURBO_NUM_CLASSES + 1];
    for (int c = 0; c < TURBO_NUM_CLASSES; ++c) {
        hbm_class[c] = !fused;
        if (fused && shape->cls_count[c]) {
            const turbo_shape_t cs = class_shape(shape, c);
            hbm_class[c] = solve_mode(&cs) == DP_SOLVE_GLOBAL;
        }
    }
    hbm_class[TURBO_NUM_CLASSES] = true;                 // long windows: always HBM planes
    int64_t total = 0;
    for (int32_t w = 0; w < shape->num_windows; ++w) {
        const turbo_window_t &win = windows_host[w];
        const int rc = std::min(row_class((int64_t)win.budget_bound + 1), TURBO_NUM_CLASSES);
        if (hbm_class[rc]) total += choice_plane_bytes(win.num_frames, win.budget_bound, win.num_exits);
    }
    *hbm_bytes = total;
    return TURBO_OK;
}

turbo_status_t turbo_mckp_solve_workspace(const turbo_shape_t *shape, size_t *bytes)
{
    if (!shape || !bytes) return TURBO_ERR_INVALID_ARG;
    *bytes = solve_needs_workspace(shape) ? (size_t)shape->workspace_bytes : 0;
    return TURBO_OK;
}

turbo_status_t turbo_mckp_solve(const turbo_shape_t *shape, const turbo_window_t *windows, const int32_t *opt_gain,
                                const int32_t *opt_cost, void *workspace, size_t workspace_bytes,
                                int32_t *best_gain, int32_t *best_cost, uint8_t *feasible, uint8_t *exit_out,
                                int64_t *status, turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!windows || !best_gain || !best_cost || !feasible || !status) return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && !exit_out) return TURBO_ERR_INVALID_ARG;
    if (shape->total_options > 0 && (!opt_gain || !opt_cost)) return TURBO_ERR_INVALID_ARG;
    if (solve_needs_workspace(shape) &&
        ((int64_t)workspace_bytes < shape->workspace_bytes || (shape->workspace_bytes > 0 && !workspace)))
        return TURBO_ERR_WORKSPACE;
    return run_dp(shape, RUN_SOLVE,
                  base_params(shape, windows, opt_gain, opt_cost, workspace, best_gain, best_cost, feasible, exit_out,
                              status),
                  stream);
}

static turbo_status_t schedule_impl(const turbo_shape_t *shape, const turbo_profile_t *profiles,
                                    turbo_window_t *windows, const uint8_t *class_id, const float *theta,
                                    float inv_width, uint8_t *class_out, const int32_t *capacity, int32_t base_cost,
                                    void *workspace, size_t workspace_bytes, int32_t *best_gain, int32_t *best_cost,
                                    uint8_t *feasible, uint8_t *exit_out, int64_t *stats, int64_t *status,
                                    turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!profiles || !windows || !best_gain || !best_cost || !feasible || !stats || !status || base_cost < 0)
        return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && (!class_id || !exit_out)) return TURBO_ERR_INVALID_ARG;
    if (solve_needs_workspace(shape) &&
        ((int64_t)workspace_bytes < shape->workspace_bytes || (shape->workspace_bytes > 0 && !workspace)))
        return TURBO_ERR_WORKSPACE;
    DpParams P = base_params(shape, windows, nullptr, nullptr, workspace, best_gain, best_cost, feasible, exit_out,
                             status);
    P.windows_rw = windows;
    P.profiles = profiles;
    P.class_id = class_id;
    P.theta = theta;
    P.inv_width = inv_width;
    P.class_out = class_out;
    P.capacity = capacity;
    P.base_cost = base_cost;
    P.fuse = 1;
    P.stats = stats;
    return run_dp(shape, RUN_SCHEDULE, P, stream);
}

turbo_status_t turbo_schedule(const turbo_shape_t *shape, const turbo_profile_t *profiles, turbo_window_t *windows,
                              const uint8_t *class_id, const int32_t *capacity, int32_t base_cost, void *workspace,
                              size_t workspace_bytes, int32_t *best_gain, int32_t *best_cost, uint8_t *feasible,
                              uint8_t *exit_out, int64_t *stats, int64_t *status, turbo_stream_t stream)
{
    return schedule_impl(shape, profiles, windows, class_id, nullptr, 0.0f, nullptr, capacity, base_cost, workspace,
                         workspace_bytes, best_gain, best_cost, feasible, exit_out, stats, status, stream);
}

turbo_status_t turbo_schedule_theta(const turbo_shape_t *shape, const turbo_profile_t *profiles,
                                    turbo_window_t *windows, const float *theta, float bucket_width,
                                    uint8_t *class_out, const int32_t *capacity, int32_t base_cost, void *workspace,
                                    size_t workspace_bytes, int32_t *best_gain, int32_t *best_cost,
                                    uint8_t *feasible, uint8_t *exit_out, int64_t *stats, int64_t *status,
                                    turbo_stream_t stream)
{
    if (!(bucket_width > 0.0f)) return TURBO_ERR_INVALID_ARG;
    if (shape && shape->total_frames > 0 && (!theta || !class_out)) return TURBO_ERR_INVALID_ARG;
    const float inv = 1.0f / bucket_width;             // rounded to float32 once, as turbo_bucketize
    return schedule_impl(shape, profiles, windows, class_out, theta, inv, class_out, capacity, base_cost, workspace,
                         workspace_bytes, best_gain, best_cost, feasible, exit_out, stats, status, stream);
}

turbo_status_t turbo_heuristic_plan(const turbo_shape_t *shape, const turbo_window_t *windows,
                                    const int32_t *opt_gain, const int32_t *opt_cost, int32_t *gain_out,
                                    int32_t *cost_out, uint8_t *feasible, uint8_t *exit_out, int32_t *steps,
                                    turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!windows || !gain_out || !cost_out || !feasible) return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && !exit_out) return TURBO_ERR_INVALID_ARG;
    if (shape->total_options > 0 && (!opt_gain || !opt_cost)) return TURBO_ERR_INVALID_ARG;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    cudaError_t e = launch_heuristic(shape, windows, opt_gain, opt_cost, gain_out, cost_out, feasible, exit_out, steps,
                                     d.num_sms, d.smem_per_cta_optin, (cudaStream_t)stream);
    if (e == cudaErrorInvalidConfiguration) {
        cudaGetLastError();
        return TURBO_ERR_UNSUPPORTED;
    }
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

// bytes of the general (R20) program's scratch for this batch: one slice per SM; 0 when the batch
// has too many frames per window for it
static int64_t batched_ws_bytes(const turbo_shape_t *s, int num_sms)
{
    // the program's last layer holds C(N + K, K) choice bytes: bounded to 2^24 (16 MB per slice)
    const int64_t N = s->max_frames, K = std::min<int32_t>(s->max_exits, 8);
    double T = 1.0;
    for (int64_t r = 0; r < K; ++r) T = T * (double)(N + K - r) / (double)(r + 1);
    if (T > (double)(1 << 24)) return 0;
    return batched_dp_bytes(s->max_frames, s->max_exits, num_sms);
}

turbo_status_t turbo_batched_workspace(const turbo_shape_t *shape, size_t *bytes)
{
    if (!shape || !bytes) return TURBO_ERR_INVALID_ARG;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    *bytes = (size_t)batched_ws_bytes(shape, d.num_sms);
    return TURBO_OK;
}

turbo_status_t turbo_batched_plan(const turbo_shape_t *shape, const turbo_window_t *windows,
                                  const turbo_profile_t *profiles, const int32_t *batch_cost, int32_t batch_cap,
                                  const uint8_t *class_id, void *workspace, size_t workspace_bytes,
                                  int32_t *best_gain, int32_t *best_cost, uint8_t *feasible, uint8_t *exit_out,
                                  int64_t *status, turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!windows || !profiles || !batch_cost || !best_gain || !best_cost || !feasible || !status)
        return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && (!class_id || !exit_out)) return TURBO_ERR_INVALID_ARG;
    if (batch_cap < 0 || batch_cap > 255 || shape->max_frames > batch_cap) return TURBO_ERR_UNSUPPORTED;
    // count vectors per window: C(N + K - 1, K - 1) at the batch maxima; counts code (N+1)^(K-1)
    const int64_t N = shape->max_frames, K = shape->max_exits;
    double vectors = 1.0, code = 1.0;
    for (int64_t r = 0; r < K - 1; ++r) {
        vectors = vectors * (double)(N + K - 1 - r) / (double)(r + 1);
        code *= (double)(N + 1);
    }
    if (vectors > (double)(1 << 26) || code >= 4.6e18) return TURBO_ERR_UNSUPPORTED;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    // the general program (windows without R19) runs only with a workspace of the documented size
    const int64_t need = batched_ws_bytes(shape, d.num_sms);
    if (workspace != nullptr && need > 0 && (int64_t)workspace_bytes < need) return TURBO_ERR_WORKSPACE;
    void *ws = (workspace != nullptr && need > 0) ? workspace : nullptr;
    const int32_t general = (g_variant & 64) ? 2 : 1;
    cudaError_t e = launch_batched(windows, shape->num_windows, profiles, batch_cost, batch_cap, class_id, best_gain,
                                   best_cost, feasible, exit_out, status, (int32_t)K, (int32_t)N, ws, general,
                                   d.num_sms, (cudaStream_t)stream);
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

turbo_status_t turbo_bucketize(const float *theta, int64_t num_frames, int32_t num_classes, float bucket_width,
                               uint8_t *class_out, turbo_stream_t stream)
{
    if (num_frames < 0 || num_classes < 1 || num_classes > 256 || !(bucket_width > 0.0f)) return TURBO_ERR_INVALID_ARG;
    if (num_frames == 0) return TURBO_OK;
    if (!theta || !class_out) return TURBO_ERR_INVALID_ARG;
    if ((reinterpret_cast<uintptr_t>(theta) & 15) || (reinterpret_cast<uintptr_t>(class_out) & 3))
        return TURBO_ERR_INVALID_ARG;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    const float inv = 1.0f / bucket_width;
    cudaError_t e = launch_bucketize(theta, num_frames, num_classes, inv, class_out, d.num_sms, (cudaStream_t)stream);
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

turbo_status_t turbo_batches(const turbo_shape_t *shape, const turbo_window_t *windows, const uint8_t *exit_out,
                             int32_t *count_out, int32_t *order_out, const int32_t *batch_cost, int32_t batch_cap,
                             int64_t *latency_out, int64_t *status, turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!windows || !count_out) return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && (!exit_out || !order_out)) return TURBO_ERR_INVALID_ARG;
    if (latency_out && (!batch_cost || !status || batch_cap < 0 || batch_cap > 65535)) return TURBO_ERR_INVALID_ARG;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    cudaError_t e = launch_batches(windows, shape->num_windows, exit_out, count_out, order_out,
                                   latency_out ? batch_cost : nullptr, batch_cap, latency_out, status, d.num_sms,
                                   (cudaStream_t)stream);
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

turbo_status_t turbo_stats(const turbo_shape_t *shape, const turbo_window_t *windows, const uint8_t *class_id,
                           const uint8_t *exit_out, const int32_t *best_gain, const int32_t *best_cost,
                           const uint8_t *feasible, int64_t *stats, turbo_stream_t stream)
{
    if (!shape) return TURBO_ERR_INVALID_ARG;
    if (shape->num_windows == 0) return TURBO_OK;
    if (!windows || !best_gain || !best_cost || !feasible || !stats) return TURBO_ERR_INVALID_ARG;
    if (shape->total_frames > 0 && (!class_id || !exit_out)) return TURBO_ERR_INVALID_ARG;
    DeviceInfo d;
    if (device_info(&d) != cudaSuccess) return TURBO_ERR_CUDA;
    cudaError_t e = launch_stats(windows, shape->num_windows, class_id, exit_out, best_gain, best_cost, feasible,
                                 stats, d.num_sms, (cudaStream_t)stream);
    return e == cudaSuccess ? TURBO_OK : TURBO_ERR_CUDA;
}

}  // extern "C"

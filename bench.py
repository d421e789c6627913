#!/usr/bin/env python
"""Benchmark of the Turbo MCKP scheduler hot path on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl turbo|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N      (N > 1, NCCL allreduce of the stats)

A step is one pass of the whole path over the rank's windows:
turbo_schedule (a1..a6 in one launch; --path solve: turbo_profile_lookup -> turbo_mckp_solve ->
turbo_stats) [-> allreduce of the int64[181] stats over NCCL when N > 1]. Inputs are generated on the
host from the seeded generator (synth/) and copied to HBM before timing. Weak scaling: each
rank plans its own windows (window ids offset by rank), per-GPU work fixed.
The metric is BASELINE.json's: DP cell-updates/s (sum over windows of N_w (B_w + 1) per
step, whole job) -- windows/s is reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MCKP DP cell-updates/s and windows/s at 1/2/4/8 B200 (% of roofline)"
UNIT = "cell-updates/s"

# per-GPU window shares (weak scaling); c3's share is its 8-GPU shard
WORKLOADS = {
    "c1": dict(config=1, per_gpu=1, desc="1 window x 30 frames, K=4, B=120"),
    "c2": dict(config=2, per_gpu=1024, desc="1024 streams x 1 s windows at 30 fps (N=30), K=5, B=1000 per GPU"),
    "c3": dict(config=3, per_gpu=8192, desc="8192 windows x 300 frames, K=8, B=4096 per GPU (c3 = 65536 over 8 GPUs)"),
    "c4": dict(config=4, per_gpu=1, desc="single long window: 3000 frames, K=6, B=2^20 (grid-spanning row; replicas)"),
    "c5": dict(config=5, per_gpu=16384, desc="mixed sweep: K 2-16, B 64-16384, N 30-300, skewed classes; "
                                           "16384 windows (the whole config) per GPU"),
    # large budgets (not a BASELINE config): a batch of long windows, each planned by one
    # thread-block cluster (dp_cluster.cu) -- c4-shaped frames and exits at 60,001 cells
    "lw": dict(config="lw", per_gpu=64, desc="64 long windows x 300 frames, K=6, B=60000 per GPU (one thread-block "
                                             "cluster per window)"),
    # NEXT-4 (batched latency): the c2 window shape with batch latency tables
    "b2": dict(config="b2", per_gpu=1024, desc="NEXT-4 batched-cost GAP: 1024 windows x 30 frames, K=5, B=1000, "
                                               "I_k(n) = ceil(c_k (2+3n)/5) per GPU"),
}
METRIC_B = "NEXT-4 exact batched-cost plans: count vectors evaluated/s (and windows/s)"
UNIT_B = "count-vectors/s"
ISSUE_PEAK = 148 * 4 * 1.965e9          # warp-instructions/s: 4 SMSPs x 1 issue/clk x sm_max_mhz
ALU_PEAK = 148 * 128 * 1.965e9          # 32-bit integer lane-operations/s: 4 SMSPs x 32 lanes per clock
ALG_OPS_PER_VECTOR = 11                 # NEXT-4 enumeration: per count vector (see the roofline note)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: run every rank on one device (the multi-rank code path on a 1-GPU box, with the
    # gloo backend -- host-staged collectives, no kernel waits on another rank)
    if os.environ.get("TURBO_BENCH_DEVICE") is not None:
        local = int(os.environ["TURBO_BENCH_DEVICE"])
    return ws, rank, local


def init_dist(torch, dist, local, backend):
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)


def make_workload(name: str, rank: int, world: int = 1, scaling: str = "weak"):
    """The rank's windows. weak: per_gpu windows at offset rank * per_gpu (per-GPU work fixed).
    strong: the config's whole window set (BASELINE.json), split into contiguous work-balanced
    ranges (shard.py) -- the same total work at every N."""
    import synth
    spec = WORKLOADS[name]
    if name.startswith("b"):
        return synth.make_batched_config(int(name[1:]), num_windows=spec["per_gpu"],
                                         window_offset=rank * spec["per_gpu"])
    if name == "lw":                   # replicas of the shape; each rank its own seeded windows
        n = spec["per_gpu"]
        return synth.concat_workloads([synth.make_long_window(500 + rank * n + s, N=300, K=6, B=60000)
                                       for s in range(n)])
    if scaling == "strong":
        from paper_2207_00172_b200.shard import shard_ranges, work_per_window
        whole = synth.CONFIGS[spec["config"]]["W"] if spec["config"] in synth.CONFIGS else 16384
        full = synth.make_config(spec["config"])
        assert full.num_windows == whole
        lo, hi = shard_ranges(work_per_window(full.num_frames, full.budget, full.num_exits), world)[rank]
        return synth.make_config(spec["config"], window_offset=lo, num_windows=hi - lo)
    return synth.make_config(spec["config"], window_offset=rank * spec["per_gpu"], num_windows=spec["per_gpu"])


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def measure_smem_peak(dev) -> dict:
    """The shared-memory roofline denominator, measured live on this GPU: the library's
    conflict-free LDS stream kernel (turbo_debug_smem_stream) on every SM, CUDA events, best of 5
    after warm-up, 1 and 2 CTAs (1024 threads) per SM, 4/8/16-byte loads per lane. The peak is the
    best over load widths (the most the pipe delivers); the 4-byte figure -- the DP's own access
    type -- is reported beside it."""
    import torch
    from paper_2207_00172_b200 import turbo
    sink = torch.zeros(4096, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    rates = {}
    for width in (4, 8, 16):
        best = 0.0
        for ctas in (1, 2):
            iters = 24000 // (ctas * width)
            for _ in range(2):
                turbo.smem_stream(iters, ctas, sink, width)
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                nbytes = turbo.smem_stream(iters, ctas, sink, width)
                e1.record(stream)
                e1.synchronize()
                best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        rates[width] = best
    return {"gbs": max(rates.values()), "gbs_by_bytes_per_lane": {str(k): v for k, v in rates.items()},
            "how": "turbo_debug_smem_stream: conflict-free ld.shared stream (4/8/16 B per lane), 1024 threads x "
                   "{1,2} CTAs per SM on every SM, CUDA events, best of 5 (burst); peak = best width"}


def _vectors(wl) -> int:
    """Count vectors per window: C(N + K - 1, K - 1), summed."""
    from math import comb
    return int(sum(comb(int(n) + int(k) - 1, int(k) - 1) for n, k in zip(wl.num_frames, wl.num_exits)))


def run_batched(args):
    """NEXT-4 leg: turbo_batched_plan on b<k> windows (device timing with CUDA graphs and L2 flush,
    e2e through the public API with host buffers, CPU oracle baseline)."""
    import torch
    import numpy as np
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        torch.cuda.set_device(local)
        init_dist(torch, dist, local, args.dist_backend)
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2207_00172_b200 import build as tbuild, turbo
    if not os.path.exists(turbo.LIB_PATH):
        tbuild.build()
    turbo.load()
    name = args.workload
    wl = make_workload(name, rank)
    b = turbo.make_batch(wl.profiles_gain, wl.profiles_cost, wl.profiles_shape, wl.num_frames, wl.budget, wl.profile,
                         class_id=wl.class_id, device=dev, with_plan_workspace=False)
    bt = turbo.batch_cost_table(wl.profiles_batch, wl.profiles_shape, wl.batch_cap, device=dev)
    W, F = wl.num_windows, wl.total_frames
    vec = _vectors(wl)

    nws = turbo.batched_workspace(b.shape)                 # the general program's scratch (R20)
    ws_t = torch.empty(max(nws, 16), dtype=torch.uint8, device=dev) if nws else None
    if args.variant:
        turbo.debug_set_variant(args.variant)             # 64: the general program on every window

    def call(stream=None):
        turbo.batched_plan(b.shape, b.windows_dev, b.profiles_dev, bt, wl.batch_cap, b.class_id, b.best_gain,
                           b.best_cost, b.feasible, b.exit_out, b.status, stream, workspace=ws_t)

    for _ in range(max(args.warmup, 3)):
        call()
    torch.cuda.synchronize(dev)
    c0 = turbo.launch_count()
    call()
    torch.cuda.synchronize(dev)
    launches = turbo.launch_count() - c0
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(3):
        g.replay()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk.start()
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        evs[k][0].record(stream)
        g.replay()
        evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    t_step = sum(a.elapsed_time(bb) for a, bb in evs) / args.steps / 1e3
    st = b.status.cpu().numpy()
    if st[0] != -1 or st[1] != -1:
        raise RuntimeError(f"status words set during bench: {st}")
    # e2e: class ids H2D from pinned host memory, the C-ABI call, results D2H (pinned)
    h_cls = torch.empty(max(F, 1), dtype=torch.uint8).pin_memory()
    h_cls[:F] = torch.as_tensor(wl.class_id)
    h_out = torch.empty_like(b.out_arena, device="cpu").pin_memory()
    for _ in range(3):
        b.class_id[:F].copy_(h_cls[:F], non_blocking=True)
        call()
        h_out.copy_(b.out_arena, non_blocking=True)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        b.class_id[:F].copy_(h_cls[:F], non_blocking=True)
        call()
        h_out.copy_(b.out_arena, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    t_e2e = e0.elapsed_time(e1) / args.steps / 1e3
    if dist is not None:
        tt = torch.tensor([t_step, t_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_e2e = float(tt[0]), float(tt[1])
    N = ws
    ops = None
    opf = os.path.join(ROOT, "profiles", f"issue_{name}.json")
    if os.path.exists(opf):
        ops = json.load(open(opf)).get("warp_instructions_per_launch")
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        import synth
        n_sub = 64
        synth_sub = synth.make_batched_config(int(name[1:]), num_windows=n_sub)
        t0 = time.time()
        reps = 0
        while time.time() - t0 < args.cpu_seconds or reps == 0:
            oracle.batched(synth_sub)
            reps += 1
        dt = time.time() - t0
        cpu = {"value": _vectors(synth_sub) * reps / dt, "unit": UNIT_B, "cores": 1, "kind": "oracle",
               "sample": f"{reps} passes over {n_sub} {name} windows (count-vector enumeration, gcc -O2, 1 thread)"}
    if rank == 0:
        line = {
            "metric": METRIC_B, "value": vec * N / t_step, "unit": UNIT_B, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (seeded splitmix64 generator, synth/; supermodular Appendix-B gains, batch latency tables)",
            "config": {"workload": f"{name}: {WORKLOADS[name]['desc']}", "windows_per_gpu": W,
                       "count_vectors_per_gpu_step": vec, "path": "turbo_batched_plan (1 launch)",
                       "l2": "flushed between timed steps (256 MiB write outside the step events)",
                       "parallelism": f"weak dp{N} (windows sharded, no collective)"},
            "windows_per_s": W * N / t_step,
            "roofline": {"bound": "alu", "achieved": vec * ALG_OPS_PER_VECTOR / t_step, "peak": ALU_PEAK,
                         "unit": "int-ops/s", "frac": vec * ALG_OPS_PER_VECTOR / t_step / ALU_PEAK,
                         "traffic": None, "kernel": "turbo::batched_kernel",
                         "note": f"achieved = count vectors x {ALG_OPS_PER_VECTOR} algorithmic integer operations "
                                 "per vector (2 batch-table reads + 2 prefix-gain reads, 2 adds for the cost, 2 subs "
                                 "+ 1 add for the gain, 1 compare against the budget, 1 against the best) / live "
                                 "launch time; peak = 148 SMs x 128 int lanes/clk x sm_max_mhz (DESIGN.md §6)",
                         "issue": {"achieved": (ops / t_step) if ops else None, "peak": ISSUE_PEAK,
                                   "unit": "warp-instructions/s", "frac": (ops / t_step / ISSUE_PEAK) if ops else None,
                                   "source": "profiles/issue_<workload>.json (ncu smsp__inst_executed per launch)"}},
            "e2e": {"value": vec * N / t_e2e, "unit": UNIT_B, "h2d_bytes_per_step": F,
                    "d2h_bytes_per_step": int(b.out_arena.numel()), "ms_per_step": t_e2e * 1e3},
            "gpu_launches": launches * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line). NVML is polled every ~1 ms from a thread, so even a
    millisecond-scale timed region gets samples; nvidia-smi (50 ms period) is the fallback."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    REASONS = (("hw_slowdown", 0x8), ("sw_power_cap", 0x4), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.samples = []              # (sm_mhz, max_mhz, reasons bitmask) from NVML
        self.running = False
        self.nvml = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = self.gpu
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.gpu < len(ids) and ids[self.gpu].isdigit():
                idx = int(ids[self.gpu])
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def start(self):
        try:
            self.nvml = self._nvml_handle()
        except Exception:
            self.nvml = None
        if self.nvml is not None:
            self.running = True
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            while not self.samples and self.thread.is_alive():
                time.sleep(0.0002)    # the first sample precedes the first timed launch
            return
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        try:
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            smax = None
        while self.running:
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), smax, int(get_reasons(h))))
            except Exception:
                break
            time.sleep(0.001)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.nvml is not None:
            self.running = False
            self.thread.join(timeout=2)
            sm = [x[0] for x in self.samples]
            smax = [x[1] for x in self.samples if x[1]]
            reasons = sorted({nm for x in self.samples for nm, bit in self.REASONS if x[2] & bit})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                    "reasons": reasons, "samples": len(sm), "source": "nvml, ~1 ms period"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi, 50 ms period"}


# ----------------------------------------------------------------------------- oracle legs
def oracle_rate(wl, budget_s: float, threads: int):
    """Oracle (as it stands) on repetitions of the workload's windows until budget_s elapsed."""
    import oracle
    og, oc, _, _ = oracle.lookup(wl)
    bud = oracle.budget(wl.capacity, wl.num_frames, wl.base_cost)
    K = wl.num_exits
    cells = wl.total_cells
    t0 = time.perf_counter()
    reps = 0
    while True:
        oracle.plan(wl.num_frames, bud, K, og, oc, "table", threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return cells * reps / el, reps, el


def sample_for_oracle(wl, max_cells: float):
    """A bounded prefix of the workload's windows (whole windows) with <= max_cells cells."""
    cells = (wl.num_frames.astype(np.int64) * (wl.budget.astype(np.int64) + 1))
    cum = np.cumsum(cells)
    n = int(np.searchsorted(cum, max_cells, side="right"))
    n = max(1, min(n, wl.num_windows))
    return wl.subset(0, n)


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return 0
    name = args.workload
    if name.startswith("b"):                     # NEXT-4: the batched oracle on a window sample
        import oracle
        import synth
        sub = synth.make_batched_config(int(name[1:]), num_windows=64)
        for _ in range(args.warmup):
            oracle.batched(sub)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.batched(sub)
        el = time.perf_counter() - t0
        value = _vectors(sub) * args.steps / el
        sample = f"64 of {WORKLOADS[name]['per_gpu']} windows of {name} per step, count-vector enumeration, 1 thread"
        print(json.dumps({"impl": "reference", "metric": METRIC_B, "value": value, "unit": UNIT_B,
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded splitmix64, synth/)",
                          "config": {"workload": f"{name}: {WORKLOADS[name]['desc']}", "oracle_sample_windows": 64},
                          "cpu_baseline": {"value": value, "unit": UNIT_B, "cores": 1, "kind": "oracle",
                                           "sample": sample},
                          "e2e": {"value": value, "unit": UNIT_B, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return 0
    wl = make_workload(name, 0)
    threads = os.cpu_count() or 1
    # each step: a bounded sample (whole windows) of ~0.15 s of oracle work on all cores
    sub = sample_for_oracle(wl, 2.0e8 * threads * 0.15)
    import oracle
    og, oc, _, _ = oracle.lookup(sub)
    bud = oracle.budget(sub.capacity, sub.num_frames, sub.base_cost)
    K = sub.num_exits
    for _ in range(args.warmup):
        oracle.plan(sub.num_frames, bud, K, og, oc, "table", threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.plan(sub.num_frames, bud, K, og, oc, "table", threads)
    el = time.perf_counter() - t0
    value = sub.total_cells * args.steps / el
    sample = (f"{sub.num_windows} of {wl.num_windows} windows of {name} per step "
              f"({sub.total_cells} cells), table DP + reconstruction, gcc -O2, {threads} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded splitmix64, synth/)",
            "config": {"workload": f"{name}: {WORKLOADS[name]['desc']}", "oracle_sample_windows": sub.num_windows},
            "windows_per_s": sub.num_windows * args.steps / el,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
TURBO_BIG_CELLS = 24576          # include/turbo.h: rows longer than this use the grid kernel


def _has_long_windows(wl) -> bool:
    return bool((wl.budget.astype(np.int64) + 1 > TURBO_BIG_CELLS).any())

def run_turbo(args):
    import torch
    ws, rank, local = dist_env()
    dist = None
    if ws > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
        torch.cuda.set_device(local)
        init_dist(torch, dist, local, args.dist_backend)
        if rank == 0:
            print(f"[bench] communicator: {dist.get_world_size()} ranks (backend {dist.get_backend()})",
                  file=sys.stderr, flush=True)
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2207_00172_b200 import build as tbuild, turbo
    if not os.path.exists(turbo.LIB_PATH):
        tbuild.build()
    turbo.load()

    if args.variant:
        turbo.debug_set_variant(args.variant)      # A/B runs only (turbo.h turbo_debug_set_variant)
    name = args.workload
    wl = make_workload(name, rank, ws, args.scaling)
    path = args.path
    if path == "auto":      # one fused launch unless long windows need the grid kernel
        path = "solve" if _has_long_windows(wl) else "schedule"
    b = turbo.batch_from_workload(wl, device=dev, with_plan_workspace=(path == "plan"))
    stream = torch.cuda.current_stream(dev)
    fused = path == "solve"
    cells = wl.total_cells
    W = wl.num_windows

    def dominant(stats_buf=None):
        sb = b.stats if stats_buf is None else stats_buf
        if path == "schedule":       # a1..a6 in one launch
            turbo.schedule(b.shape, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost, b.solve_ws,
                           b.best_gain, b.best_cost, b.feasible, b.exit_out, sb, b.status)
        elif path == "solve":
            turbo.mckp_solve(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, b.solve_ws, b.best_gain,
                             b.best_cost, b.feasible, b.exit_out, b.status)
        else:
            turbo.mckp_plan(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, b.workspace, b.best_gain,
                            b.best_cost, b.feasible, b.status)

    def step(reset: bool = True, stats_buf=None):
        """One pass of the path. stats_buf: accumulate a6 into this buffer instead of the arena's
        (the second buffer of the overlapped allreduce, N > 1)."""
        stream = torch.cuda.current_stream(dev)
        sb = b.stats if stats_buf is None else stats_buf
        if reset:                    # stats = 0, status = -1: one device-to-device copy
            if stats_buf is None:
                turbo.reset_outputs(b)
            else:
                stats_buf.zero_()
                b.status.fill_(-1)
        if path == "schedule":
            dominant(stats_buf)
            return
        turbo.profile_lookup(b.shape, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost,
                             b.opt_gain, b.opt_cost, b.status, stream)
        if fused:
            turbo.mckp_solve(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, b.solve_ws, b.best_gain, b.best_cost,
                             b.feasible, b.exit_out, b.status, stream)
        else:
            turbo.mckp_plan(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, b.workspace, b.best_gain, b.best_cost,
                            b.feasible, b.status, stream)
        if not fused:
            turbo.backtrack(b.shape, b.windows_dev, b.opt_cost, b.workspace, b.best_cost, b.feasible, b.exit_out,
                            stream)
        turbo.stats(b.shape, b.windows_dev, b.class_id, b.exit_out, b.best_gain, b.best_cost, b.feasible, sb,
                    stream)
    # L2 flush buffer (> 126 MB L2) written between timed steps (outside the timed events)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    for _ in range(max(args.warmup, 3)):
        step()
        if dist is not None:
            dist.all_reduce(b.stats)
    torch.cuda.synchronize(dev)
    # kernels one step launches, counted by the library itself (turbo_launch_count)
    c0 = turbo.launch_count()
    step()
    torch.cuda.synchronize(dev)
    launches_per_step = turbo.launch_count() - c0
    c0 = turbo.launch_count()
    dominant()
    torch.cuda.synchronize(dev)
    launches_dominant = turbo.launch_count() - c0

    # The step's kernels are captured once into a CUDA graph (launch latency off the device
    # timeline; the same C-ABI launches, replayed); the NCCL allreduce stays eager.
    g_step = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_step):
        step()
    # N > 1: the a6 allreduce of step k runs on a communication stream while step k+1 computes, so
    # the statistics are double-buffered (step k+2 reuses step k's buffer only after its allreduce
    # completed -- that wait is inside step k+2's timed window); the last step's allreduce is
    # waited for inside the last window
    stats2 = torch.zeros_like(b.stats)
    g_step2 = None
    comm = None
    if dist is not None:
        step(stats_buf=stats2)
        dist.all_reduce(stats2)
        torch.cuda.synchronize(dev)
        g_step2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_step2):
            step(stats_buf=stats2)
        comm = torch.cuda.Stream(device=dev)
    g_dp = torch.cuda.CUDAGraph()                        # the dominant kernel alone
    with torch.cuda.graph(g_dp):
        dominant()
    stream = torch.cuda.current_stream(dev)
    for _ in range(3):
        g_step.replay()
        g_dp.replay()
    torch.cuda.synchronize(dev)

    g_lk = torch.cuda.CUDAGraph()                        # a2 gather alone (HBM roofline)
    with torch.cuda.graph(g_lk):
        turbo.profile_lookup(b.shape, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost,
                             b.opt_gain, b.opt_cost, b.status)
    for _ in range(3):
        g_lk.replay()
    torch.cuda.synchronize(dev)
    turbo.reset_outputs(b)

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    evd = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    evl = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk.start()
    ev_ar = [torch.cuda.Event(), torch.cuda.Event()]
    ar_pending = [False, False]
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        evs[k][0].record(stream)
        if dist is None:
            g_step.replay()
        else:
            j = k & 1
            if ar_pending[j]:
                stream.wait_event(ev_ar[j])              # this buffer's previous allreduce is done
            (g_step if j == 0 else g_step2).replay()
            done = torch.cuda.Event()
            done.record(stream)
            comm.wait_event(done)
            with torch.cuda.stream(comm):
                dist.all_reduce(b.stats if j == 0 else stats2)
            ev_ar[j].record(comm)
            ar_pending[j] = True
            if k == args.steps - 1:
                stream.wait_event(ev_ar[j])              # the last allreduce inside the last window
        evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        evd[k][0].record(stream)
        g_dp.replay()
        evd[k][1].record(stream)
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        evl[k][0].record(stream)
        g_lk.replay()
        evl[k][1].record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    t_step = sum(a.elapsed_time(bb) for a, bb in evs) / args.steps / 1e3          # s per step (this rank)
    t_dp = sum(a.elapsed_time(bb) for a, bb in evd) / args.steps / 1e3
    per_step = sorted(a.elapsed_time(bb) for a, bb in evs)                          # ms, this rank
    per_dp = sorted(a.elapsed_time(bb) for a, bb in evd)
    t_lk = sum(a.elapsed_time(bb) for a, bb in evl) / args.steps / 1e3
    # correctness of the timed run (cheap, rank-local): no status errors (checked BEFORE the reset;
    # the lookup graph leaves status untouched on valid inputs)
    st = b.status.cpu().numpy()
    if st[0] != -1 or st[1] != -1:
        raise RuntimeError(f"status words set during bench: {st}")
    turbo.reset_outputs(b)

    # ---- e2e through the C ABI with HOST buffers (pinned), H2D inputs + D2H results inside
    F = int(b.shape.total_frames)
    # host buffers (pinned) mirroring the device input / output arenas: one copy each way
    turbo.reset_outputs(b)           # the host input image carries the initial stats / status
    h_in = torch.empty_like(b.in_arena, device="cpu").pin_memory()
    h_in.copy_(b.in_arena)
    h_out = torch.empty_like(b.out_arena, device="cpu").pin_memory()
    h2d = b.in_arena.numel()
    d2h = b.out_arena.numel()

    def e2e_step_eager():
        # the public API, called eagerly (no graph): H2D inputs, the C-ABI calls, D2H results
        b.in_arena.copy_(h_in, non_blocking=True)     # inputs + initial stats/status
        step(reset=False)
        if dist is not None:
            dist.all_reduce(b.stats)
        h_out.copy_(b.out_arena, non_blocking=True)

    # the serving form: the same H2D copy, C-ABI call(s) and D2H copy captured ONCE into a CUDA graph
    # and replayed every step (the copies still move every byte every step; the graph removes the
    # host launch gaps between copy engine and SMs). N > 1: the allreduce stays eager between the
    # two graphs.
    for _ in range(3):
        e2e_step_eager()
    torch.cuda.synchronize(dev)
    g_e2e_a = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_e2e_a):
        b.in_arena.copy_(h_in, non_blocking=True)
        step(reset=False)
        if dist is None:
            h_out.copy_(b.out_arena, non_blocking=True)
    g_e2e_b = None
    if dist is not None:
        g_e2e_b = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_e2e_b):
            h_out.copy_(b.out_arena, non_blocking=True)

    def e2e_step_graph():
        g_e2e_a.replay()
        if dist is not None:
            dist.all_reduce(b.stats)
            g_e2e_b.replay()

    # the same graph with the two copies done by the SMs (turbo_memcpy_sm over mapped pinned memory)
    g_sm_a = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_sm_a):
        turbo.memcpy_sm(b.in_arena, h_in)
        step(reset=False)
        if dist is None:
            turbo.memcpy_sm(h_out, b.out_arena)
    g_sm_b = None
    if dist is not None:
        g_sm_b = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_sm_b):
            turbo.memcpy_sm(h_out, b.out_arena)

    def e2e_step_sm():
        g_sm_a.replay()
        if dist is not None:
            dist.all_reduce(b.stats)
            g_sm_b.replay()

    e2e_steps = max(1, min(args.steps, 50))

    def time_e2e(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        eve = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
        if dist is not None:
            dist.barrier()
        for k in range(e2e_steps):
            flush.fill_(k & 0xff)
            eve[k][0].record(stream)
            fn()
            eve[k][1].record(stream)
        torch.cuda.synchronize(dev)
        return sum(a.elapsed_time(bb) for a, bb in eve) / e2e_steps / 1e3

    # the serving form copies with the SMs when a step moves <= 1 MB (there a copy engine's fixed
    # latency dominates: c2 55.4 -> 46.7 us per step on the same box) and with the copy engines above
    sm_copies = h2d + d2h <= (1 << 20)
    t_e2e_eager = time_e2e(e2e_step_eager)
    if sm_copies:
        t_e2e_ce = time_e2e(e2e_step_graph)
        t_e2e = time_e2e(e2e_step_sm)         # last: the parity check below reads this run's outputs
    else:
        t_e2e_sm = time_e2e(e2e_step_sm)
        t_e2e = t_e2e_ce = time_e2e(e2e_step_graph)
    h_chk = h_out.clone()                     # the host copy of the results must equal the device arena
    if not torch.equal(h_chk, b.out_arena.cpu()):
        raise RuntimeError("e2e: host results differ from the device arena")

    # ---- max over ranks
    if dist is not None:
        tt = torch.tensor([t_step, t_dp, t_e2e, t_e2e_eager, t_e2e_ce], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_dp, t_e2e, t_e2e_eager, t_e2e_ce = tt.tolist()
    N = ws
    if dist is not None:           # whole-job totals (strong-scaling shards differ in size)
        tot = torch.tensor([cells, W], dtype=torch.float64, device=dev)
        dist.all_reduce(tot)
        total_cells, W_total = int(tot[0].item()), int(tot[1].item())
    else:
        total_cells, W_total = cells, W
    value = total_cells / t_step

    # ---- roofline of the dominant kernel (the DP): shared-memory bound, against the MEASURED
    # smem stream rate of this GPU (derived 148 x 128 B/clk x sm_max_mhz kept beside it)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    smem_derived = nsm * 128 * sm_max * 1e6 / 1e9                # GB/s: 32 banks x 4 B per clock per SM
    smem_meas = measure_smem_peak(dev)
    smem_peak = smem_meas["gbs"]
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s (profiling guide)"
    Kw = wl.num_exits.astype(np.int64)
    # HBM streams: the a2 gather (class ids in, option tables out, window records) and the
    # choice planes the timed call writes to HBM (0 when they stay in shared memory)
    F = int(b.shape.total_frames)
    lk_bytes = int((wl.num_frames.astype(np.int64) * (1 + 8 * Kw)).sum()) + 48 * W + 4 * W
    plane_bytes = turbo.mckp_plane_bytes(b.shape, b.windows_host, path != "plan")
    alg_bytes = int((wl.num_frames.astype(np.int64) * (wl.budget.astype(np.int64) + 1) * (4 * Kw + 4)).sum())
    achieved = alg_bytes / t_dp / 1e9
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{name}.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "int32", "data": "synthetic (seeded splitmix64 generator, synth/; paper-calibrated profiles)",
        "config": {"workload": f"{name}: {WORKLOADS[name]['desc']}", "windows_per_gpu": W,
                   "cells_per_gpu_step": cells, "path": {"schedule": "turbo_schedule (a1-a6 in one launch)", "solve": "lookup + solve (a3-a5 fused) + stats",
                            "plan": "lookup + plan + backtrack + stats"}[path],
                   "l2": "flushed between timed steps (256 MiB write outside the step events)",
                   "parallelism": f"{args.scaling} dp{N} (windows sharded, NCCL allreduce of stats)",
                   "nccl_ranks": (dist.get_world_size() if dist is not None else 1),
                   "windows_total": W_total,
                   "stats_reset": "every step, one device copy in front of the kernel (inside the step graph)"},
        "windows_per_s": W_total / t_step,
        "dp_ms": t_dp * 1e3,
        "step_ms_stats": {"median": statistics.median(per_step), "min": per_step[0], "max": per_step[-1],
                          "dp_median": statistics.median(per_dp), "dp_min": per_dp[0],
                          "note": "rank 0's per-step CUDA-event times; value/ms_per_step use the mean (max over ranks)"},
        "dp_cell_updates_per_s": total_cells / t_dp,
        "roofline": {"bound": "smem", "achieved": achieved, "peak": smem_peak, "unit": "GB/s",
                     "frac": achieved / smem_peak, "traffic": traffic,
                     "peak_source": "measured live (" + smem_meas["how"] + ")",
                     "peak_by_bytes_per_lane": smem_meas["gbs_by_bytes_per_lane"],
                     "frac_of_lds32_stream": achieved / smem_meas["gbs_by_bytes_per_lane"]["4"],
                     "peak_derived": smem_derived, "frac_of_derived": achieved / smem_derived,
                     "kernel": ("turbo::dp_cta_kernel (" + {"schedule": "turbo_schedule", "solve": "turbo_mckp_solve",
                                                            "plan": "turbo_mckp_plan"}[path] + ")"
                                + (f"; timed as the whole call, {launches_dominant} launches (DP per row class,"
                                   " walks of HBM planes, long-window grid kernel)" if launches_dominant > 1 else "")),
                     "note": "algorithmic smem bytes = cells x (4K+4) per launch (SURVEY.md 8(d)); "
                             "peak = measured smem stream rate; peak_derived = SMs x 128 B/clk x sm_max_mhz"},
        "hbm": {"peak": hbm_peak, "unit": "GB/s", "peak_source": hbm_src,
                "lookup": {"kernel": "turbo::lookup_kernel (turbo_profile_lookup, timed alone)",
                           "bytes": lk_bytes, "ms": t_lk * 1e3, "achieved": lk_bytes / t_lk / 1e9,
                           "frac": lk_bytes / t_lk / 1e9 / hbm_peak,
                           "note": "bytes = sum_w N_w (1 + 8 K_w) + 52 W (class ids, int32 option tables, "
                                   "window records + capacity); not on the timed path of turbo_schedule"},
                "choice_planes": {"bytes": plane_bytes, "achieved": plane_bytes / t_dp / 1e9,
                                  "frac": plane_bytes / t_dp / 1e9 / hbm_peak,
                                  "note": "choice planes the timed DP call writes to HBM (turbo_mckp_plane_bytes) "
                                          "over the DP call's time"}},
        "e2e": {"value": total_cells / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": t_e2e * 1e3,
                "mode": "every step: H2D of the inputs from pinned host memory, the C-ABI call(s), D2H of the "
                        "results to pinned host memory, captured once as a CUDA graph and replayed (serving "
                        "form); the copies " + ("by the SMs (turbo_memcpy_sm; <= 1 MB per step)" if sm_copies
                                                else "by the copy engines (> 1 MB per step)"),
                "copy_engine": {"value": total_cells / t_e2e_ce, "ms_per_step": t_e2e_ce * 1e3,
                                "note": "the graph with cudaMemcpyAsync copies (copy engines)"},
                "sm_copies": {"value": total_cells / (t_e2e if sm_copies else t_e2e_sm),
                              "ms_per_step": (t_e2e if sm_copies else t_e2e_sm) * 1e3,
                              "note": "the graph with turbo_memcpy_sm copies (SMs over mapped pinned memory)"},
                "eager": {"value": total_cells / t_e2e_eager, "ms_per_step": t_e2e_eager * 1e3,
                          "note": "copy-engine copies and calls issued eagerly from Python each step"}},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }
    if rank == 0 and not args.no_cpu_baseline:
        nthr = os.cpu_count() or 1
        sub = sample_for_oracle(wl, 2.5e8 * nthr * args.cpu_seconds / 10.0)
        # the timed run's own outputs (last e2e step) against the oracle on the same sample windows
        import oracle
        want = oracle.run(sub, threads=nthr)
        got = turbo.results(b)
        n_s, f_s = sub.num_windows, sub.total_frames
        bad_w = int(((got["best_gain"][:n_s].astype(np.int64) != want["best_gain"]) |
                     (got["best_cost"][:n_s].astype(np.int64) != want["best_cost"]) |
                     (got["feasible"][:n_s] != want["feasible"])).sum())
        bad_x = int((got["exits"][:f_s] != want["exits"]).sum())
        line["parity"] = {"windows_checked": n_s, "window_mismatches": bad_w, "frames_checked": f_s,
                          "exit_mismatches": bad_x,
                          "note": "outputs of the timed run (last e2e step) vs the CPU oracle on the cpu_baseline "
                                  "sample windows; the full parity suite is pytest -m gpu"}
        rate, reps, el = oracle_rate(sub, args.cpu_seconds, nthr)
        sub1 = sample_for_oracle(wl, 2.5e8 * args.cpu_seconds / 20.0)
        rate1, reps1, el1 = oracle_rate(sub1, args.cpu_seconds / 2.0, 1)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": nthr, "kind": "oracle",
                                "value_1core": rate1, "cpu_model": cpu_model(),
                                "sample": f"all cores: {reps} passes over {sub.num_windows} of the rank-0 {name} windows "
                                          f"({sub.total_cells} cells per pass), {el:.1f} s, {nthr} threads; "
                                          f"1 core: {reps1} passes over {sub1.num_windows} windows "
                                          f"({sub1.total_cells} cells), {el1:.1f} s; table DP + reconstruction, "
                                          f"gcc -O2"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["turbo", "reference"], default="turbo")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--path", choices=["auto", "schedule", "solve", "plan"], default="auto",
                    help="auto: schedule unless long windows; schedule: one fused a1..a6 launch; solve: lookup, "
                         "solve, stats; plan: 4 launches")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: per-GPU windows fixed (per_gpu of the workload); strong: the config's whole "
                         "window set split over the ranks by work (shard.py)")
    ap.add_argument("--variant", type=int, default=0, help="kernel-variant debug switch (A/B runs; 0 = automatic)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="N > 1 collective backend (gloo only to exercise the multi-rank path on one GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload.startswith("b"):
        return run_batched(args)
    return run_turbo(args)


if __name__ == "__main__":
    sys.exit(main())

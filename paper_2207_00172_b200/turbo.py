"""Thin ctypes binding of libturbo.so (include/turbo.h). Argument marshalling only.

PyTorch is used for device memory and streams (tensor.data_ptr(), the current CUDA
stream); every step of the hot path runs in the library's sm_100a kernels. There is no
CPU fallback: if the library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# TURBO_LIB selects another build of the same library (the bounds-checked checked/libturbo.so)
LIB_PATH = os.environ.get("TURBO_LIB") or os.path.join(_PKG, "libturbo.so")

TURBO_OK = 0
STATUS_NAMES = {0: "ok", 1: "invalid argument", 2: "value out of range", 3: "workspace too small",
                4: "CUDA error", 5: "unsupported shape"}
STATS_WORDS = 181
STATUS_WORDS = 2


class TurboError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed: {STATUS_NAMES.get(code, code)} ({code})")
        self.code = code


class Profile(ctypes.Structure):
    _fields_ = [("num_classes", ctypes.c_int32), ("num_exits", ctypes.c_int32),
                ("gain", ctypes.c_void_p), ("cost", ctypes.c_void_p)]


class Window(ctypes.Structure):
    _fields_ = [("first_frame", ctypes.c_int64), ("first_option", ctypes.c_int64),
                ("choice_offset", ctypes.c_int64), ("num_frames", ctypes.c_int32),
                ("budget", ctypes.c_int32), ("profile", ctypes.c_int32), ("num_exits", ctypes.c_int32),
                ("budget_bound", ctypes.c_int32), ("order", ctypes.c_int32)]


class Shape(ctypes.Structure):
    _fields_ = [("num_windows", ctypes.c_int32), ("num_profiles", ctypes.c_int32),
                ("max_frames", ctypes.c_int32), ("max_budget", ctypes.c_int32),
                ("min_exits", ctypes.c_int32), ("max_exits", ctypes.c_int32),
                ("num_classes_max", ctypes.c_int32), ("max_options", ctypes.c_int32),
                ("total_frames", ctypes.c_int64), ("total_options", ctypes.c_int64),
                ("total_cells", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("max_budget_small", ctypes.c_int32), ("num_big", ctypes.c_int32),
                ("grid_scratch_offset", ctypes.c_int64), ("ordered", ctypes.c_int32), ("cls_order", ctypes.c_int32),
                ("reserved3", ctypes.c_int64),
                ("cls_count", ctypes.c_int32 * 4), ("cls_max_budget", ctypes.c_int32 * 4),
                ("cls_max_frames", ctypes.c_int32 * 4), ("cls_max_options", ctypes.c_int32 * 4),
                ("cls_min_exits", ctypes.c_int32 * 4), ("cls_max_exits", ctypes.c_int32 * 4)]


assert ctypes.sizeof(Window) == 48
WINDOW_DTYPE = np.dtype([("first_frame", "<i8"), ("first_option", "<i8"), ("choice_offset", "<i8"),
                         ("num_frames", "<i4"), ("budget", "<i4"), ("profile", "<i4"), ("num_exits", "<i4"),
                         ("budget_bound", "<i4"), ("order", "<i4")])
assert WINDOW_DTYPE.itemsize == 48

EXPORTS = ["turbo_mckp_workspace", "turbo_profile_lookup", "turbo_mckp_plan", "turbo_backtrack",
           "turbo_mckp_solve", "turbo_mckp_solve_workspace", "turbo_mckp_plane_bytes", "turbo_schedule",
           "turbo_schedule_theta", "turbo_heuristic_plan", "turbo_stats",
           "turbo_bucketize", "turbo_batches", "turbo_batched_plan", "turbo_batched_workspace",
           "turbo_debug_set_variant", "turbo_debug_trace", "turbo_debug_u16_counter", "turbo_debug_smem_stream", "turbo_debug_tcheck_selftest",
           "turbo_launch_count", "turbo_memcpy_sm",
           "turbo_status_string", "turbo_abi_version"]

_lib = None


def load(path: Optional[str] = None):
    """Load libturbo.so (raises if absent: there is no fallback path)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"libturbo.so not built at {p}; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(p)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    lib.turbo_mckp_workspace.argtypes = [vp, i32, vp, i32, vp]
    lib.turbo_profile_lookup.argtypes = [vp, vp, vp, vp, vp, i32, vp, vp, vp, vp]
    lib.turbo_mckp_plan.argtypes = [vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp]
    lib.turbo_backtrack.argtypes = [vp, vp, vp, vp, sz, vp, vp, vp, vp]
    lib.turbo_mckp_solve.argtypes = [vp, vp, vp, vp, vp, sz, vp, vp, vp, vp, vp, vp]
    lib.turbo_mckp_solve_workspace.argtypes = [vp, vp]
    lib.turbo_mckp_plane_bytes.argtypes = [vp, vp, i32, vp]
    lib.turbo_stats.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.turbo_schedule.argtypes = [vp, vp, vp, vp, vp, i32, vp, sz, vp, vp, vp, vp, vp, vp, vp]
    lib.turbo_schedule_theta.argtypes = [vp, vp, vp, vp, ctypes.c_float, vp, vp, i32, vp, sz, vp, vp, vp, vp, vp, vp,
                                         vp]
    lib.turbo_heuristic_plan.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.turbo_bucketize.argtypes = [vp, i64, i32, ctypes.c_float, vp, vp]
    lib.turbo_batches.argtypes = [vp, vp, vp, vp, vp, vp, i32, vp, vp, vp]
    lib.turbo_batched_plan.argtypes = [vp, vp, vp, vp, i32, vp, vp, sz, vp, vp, vp, vp, vp, vp]
    lib.turbo_batched_workspace.argtypes = [vp, vp]
    lib.turbo_debug_set_variant.argtypes = [i32]
    lib.turbo_debug_trace.argtypes = [vp, i64]
    lib.turbo_debug_u16_counter.argtypes = [vp]
    lib.turbo_debug_smem_stream.argtypes = [i32, i32, i32, vp, vp, vp]
    lib.turbo_debug_tcheck_selftest.argtypes = [vp]
    lib.turbo_launch_count.argtypes = []
    lib.turbo_memcpy_sm.argtypes = [vp, vp, sz, vp]
    lib.turbo_launch_count.restype = i64
    lib.turbo_status_string.restype = ctypes.c_char_p
    lib.turbo_abi_version.restype = i32
    for name in EXPORTS:
        getattr(lib, name)
    if path is None:
        _lib = lib
    return lib


def _check(fn: str, code: int):
    if code != TURBO_OK:
        raise TurboError(fn, code)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


# ----------------------------------------------------------------------------- C-ABI mirrors
def mckp_workspace(profiles_host: Sequence[Profile], windows_host: np.ndarray) -> Shape:
    """Host-only sizing; fills the layout fields of windows_host (structured WINDOW_DTYPE array)."""
    lib = load()
    P = len(profiles_host)
    parr = (Profile * max(P, 1))(*profiles_host)
    shape = Shape()
    assert windows_host.dtype == WINDOW_DTYPE and windows_host.flags.c_contiguous
    _check("turbo_mckp_workspace",
           lib.turbo_mckp_workspace(ctypes.addressof(parr), P, windows_host.ctypes.data, len(windows_host),
                                    ctypes.addressof(shape)))
    return shape


def profile_lookup(shape, profiles_dev, windows_dev, class_id, capacity, base_cost, opt_gain, opt_cost,
                   status, stream=None):
    _check("turbo_profile_lookup",
           load().turbo_profile_lookup(ctypes.addressof(shape), _ptr(profiles_dev), _ptr(windows_dev),
                                       _ptr(class_id), _ptr(capacity), int(base_cost), _ptr(opt_gain),
                                       _ptr(opt_cost), _ptr(status), _stream(stream)))


def mckp_plan(shape, windows_dev, opt_gain, opt_cost, workspace, best_gain, best_cost, feasible, status,
              stream=None):
    nbytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check("turbo_mckp_plan",
           load().turbo_mckp_plan(ctypes.addressof(shape), _ptr(windows_dev), _ptr(opt_gain), _ptr(opt_cost),
                                  _ptr(workspace), nbytes, _ptr(best_gain), _ptr(best_cost), _ptr(feasible),
                                  _ptr(status), _stream(stream)))


def backtrack(shape, windows_dev, opt_cost, workspace, best_cost, feasible, exit_out, stream=None):
    nbytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check("turbo_backtrack",
           load().turbo_backtrack(ctypes.addressof(shape), _ptr(windows_dev), _ptr(opt_cost), _ptr(workspace),
                                  nbytes, _ptr(best_cost), _ptr(feasible), _ptr(exit_out), _stream(stream)))


def mckp_solve_workspace(shape) -> int:
    out = ctypes.c_size_t(0)
    _check("turbo_mckp_solve_workspace",
           load().turbo_mckp_solve_workspace(ctypes.addressof(shape), ctypes.addressof(out)))
    return int(out.value)


def mckp_plane_bytes(shape, windows_host: np.ndarray, fused: bool) -> int:
    """Choice-plane bytes one call writes to HBM (turbo.h turbo_mckp_plane_bytes; host only)."""
    out = ctypes.c_int64(0)
    _check("turbo_mckp_plane_bytes",
           load().turbo_mckp_plane_bytes(ctypes.addressof(shape), windows_host.ctypes.data, int(bool(fused)),
                                         ctypes.addressof(out)))
    return int(out.value)


def mckp_solve(shape, windows_dev, opt_gain, opt_cost, workspace, best_gain, best_cost, feasible, exit_out,
               status, stream=None):
    nbytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check("turbo_mckp_solve",
           load().turbo_mckp_solve(ctypes.addressof(shape), _ptr(windows_dev), _ptr(opt_gain), _ptr(opt_cost),
                                   _ptr(workspace), nbytes, _ptr(best_gain), _ptr(best_cost), _ptr(feasible),
                                   _ptr(exit_out), _ptr(status), _stream(stream)))


def schedule(shape, profiles_dev, windows_dev, class_id, capacity, base_cost, workspace, best_gain, best_cost,
             feasible, exit_out, stats_out, status, stream=None):
    nbytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check("turbo_schedule",
           load().turbo_schedule(ctypes.addressof(shape), _ptr(profiles_dev), _ptr(windows_dev), _ptr(class_id),
                                 _ptr(capacity), int(base_cost), _ptr(workspace), nbytes, _ptr(best_gain),
                                 _ptr(best_cost), _ptr(feasible), _ptr(exit_out), _ptr(stats_out), _ptr(status),
                                 _stream(stream)))


def schedule_theta(shape, profiles_dev, windows_dev, theta, bucket_width, class_out, capacity, base_cost, workspace,
                   best_gain, best_cost, feasible, exit_out, stats_out, status, stream=None):
    """NEXT-3 fused: turbo_schedule on difficulty scores (float32, device); classes written to class_out."""
    nbytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check("turbo_schedule_theta",
           load().turbo_schedule_theta(ctypes.addressof(shape), _ptr(profiles_dev), _ptr(windows_dev), _ptr(theta),
                                       float(bucket_width), _ptr(class_out), _ptr(capacity), int(base_cost),
                                       _ptr(workspace), nbytes, _ptr(best_gain), _ptr(best_cost), _ptr(feasible),
                                       _ptr(exit_out), _ptr(stats_out), _ptr(status), _stream(stream)))


def heuristic_plan(shape, windows_dev, opt_gain, opt_cost, gain_out, cost_out, feasible, exit_out, steps=None,
                   stream=None):
    """NEXT-1: the paper's prune-and-search heuristic on the option tables (comparison arm)."""
    _check("turbo_heuristic_plan",
           load().turbo_heuristic_plan(ctypes.addressof(shape), _ptr(windows_dev), _ptr(opt_gain), _ptr(opt_cost),
                                       _ptr(gain_out), _ptr(cost_out), _ptr(feasible), _ptr(exit_out), _ptr(steps),
                                       _stream(stream)))


def batched_workspace(shape) -> int:
    """Device bytes turbo_batched_plan needs for windows without R19 (turbo.h turbo_batched_workspace)."""
    out = ctypes.c_size_t(0)
    _check("turbo_batched_workspace", load().turbo_batched_workspace(ctypes.addressof(shape), ctypes.addressof(out)))
    return int(out.value)


def batched_plan(shape, windows_dev, profiles_dev, batch_cost, batch_cap, class_id, best_gain, best_cost, feasible,
                 exit_out, status, stream=None, workspace=None):
    """NEXT-4: exact plans under the batched latency tables (turbo.h turbo_batched_plan); with a
    workspace (batched_workspace bytes) also for gains without R19."""
    nbytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _check("turbo_batched_plan",
           load().turbo_batched_plan(ctypes.addressof(shape), _ptr(windows_dev), _ptr(profiles_dev), _ptr(batch_cost),
                                     int(batch_cap), _ptr(class_id), _ptr(workspace), nbytes, _ptr(best_gain),
                                     _ptr(best_cost), _ptr(feasible), _ptr(exit_out), _ptr(status), _stream(stream)))


def batch_cost_table(profiles_batch, profiles_shape, cap: int, device="cuda"):
    """Device layout of the batch latency tables: profile p at p * 16 * (cap + 1), row k = I_k(0..cap)."""
    import torch
    P = len(profiles_batch)
    t = np.zeros((max(P, 1), 16, cap + 1), dtype=np.int32)
    for p, (tab, (C, K)) in enumerate(zip(profiles_batch, profiles_shape)):
        t[p, :K] = np.asarray(tab, dtype=np.int32).reshape(K, cap + 1)
    return torch.as_tensor(t.reshape(-1), device=device)


def bucketize(theta, class_out, num_classes: int = 10, bucket_width: float = 0.1, stream=None):
    """NEXT-3: difficulty score (float32, device) -> class id (u8, device)."""
    _check("turbo_bucketize",
           load().turbo_bucketize(_ptr(theta), int(theta.numel()), int(num_classes), float(bucket_width),
                                  _ptr(class_out), _stream(stream)))


def batches(shape, windows_dev, exit_out, count_out, order_out, batch_cost=None, batch_cap=0, latency_out=None,
            status=None, stream=None):
    """NEXT-2: plan -> per-exit batch sizes [W, 16], stable per-exit frame order and (with batch_cost
    and latency_out) the executed latency sum_k I_k(n_k) per window."""
    _check("turbo_batches",
           load().turbo_batches(ctypes.addressof(shape), _ptr(windows_dev), _ptr(exit_out), _ptr(count_out),
                                _ptr(order_out), _ptr(batch_cost), int(batch_cap), _ptr(latency_out), _ptr(status),
                                _stream(stream)))


def stats(shape, windows_dev, class_id, exit_out, best_gain, best_cost, feasible, stats_out, stream=None):
    _check("turbo_stats",
           load().turbo_stats(ctypes.addressof(shape), _ptr(windows_dev), _ptr(class_id), _ptr(exit_out),
                              _ptr(best_gain), _ptr(best_cost), _ptr(feasible), _ptr(stats_out), _stream(stream)))


def debug_set_variant(v: int):
    _check("turbo_debug_set_variant", load().turbo_debug_set_variant(int(v)))


def smem_stream(iters: int, ctas_per_sm: int, sink, bytes_per_lane: int = 4, stream=None) -> float:
    """Launch the shared-memory stream kernel (turbo.h turbo_debug_smem_stream); returns the bytes
    it reads (the caller times the launch)."""
    out = ctypes.c_double(0.0)
    _check("turbo_debug_smem_stream",
           load().turbo_debug_smem_stream(int(iters), int(ctas_per_sm), int(bytes_per_lane), _ptr(sink),
                                          ctypes.addressof(out), _stream(stream)))
    return float(out.value)


def launch_count() -> int:
    """Kernels libturbo has launched so far in this process (turbo.h turbo_launch_count)."""
    return int(load().turbo_launch_count())


def debug_trace(buf=None):
    """Per-CTA phase timestamps of the DP kernels into `buf` (int64 device tensor, zeroed by the
    caller; see turbo.h turbo_debug_trace); None disables."""
    if buf is None:
        _check("turbo_debug_trace", load().turbo_debug_trace(None, 0))
    else:
        _check("turbo_debug_trace", load().turbo_debug_trace(ctypes.c_void_p(buf.data_ptr()), int(buf.numel())))


def memcpy_sm(dst, src, stream=None):
    """dst <- src (same byte size) copied by the SMs (turbo.h turbo_memcpy_sm): device tensors or
    pinned host tensors (pin_memory), e.g. a serving step's inputs and results."""
    n = dst.numel() * dst.element_size()
    if src.numel() * src.element_size() != n:
        raise ValueError("memcpy_sm: size mismatch")
    _check("turbo_memcpy_sm", load().turbo_memcpy_sm(_ptr(dst), _ptr(src), n, _stream(stream)))


def debug_u16_counter(buf=None):
    """Count the windows the DP kernels plan on u16 rows (NEXT-5) into `buf` (one-element int64
    device tensor, zeroed by the caller; turbo.h turbo_debug_u16_counter); None disables."""
    _check("turbo_debug_u16_counter",
           load().turbo_debug_u16_counter(None if buf is None else ctypes.c_void_p(buf.data_ptr())))


# ----------------------------------------------------------------------------- planner object
@dataclass
class Batch:
    """Device-resident buffers of one window batch (inputs and outputs of the hot path)."""
    shape: Shape
    windows_host: np.ndarray
    profiles_host: list
    profile_tensors: list
    profiles_dev: object
    windows_dev: object
    class_id: object
    capacity: object
    base_cost: int
    opt_gain: object
    opt_cost: object
    workspace: object
    best_gain: object
    best_cost: object
    feasible: object
    exit_out: object
    status: object
    stats: object
    solve_ws: object
    in_arena: object = None      # [capacity | class_id | stats | status] (one H2D per step)
    out_arena: object = None     # [stats | status | best_gain | best_cost | feasible | exit_out] (one D2H)
    reset: object = None         # device copy of the initial [stats = 0 | status = -1] (one D2D reset)


def _reset_template(arena, offs):
    """Initial [stats | status] bytes (zeros, then -1) on the device: one D2D copy resets both."""
    t = arena[offs[2]: offs[4]].clone()
    t.view(-1)[:] = 0
    t[offs[3] - offs[2]:].view(-1).fill_(255)      # status int64 = -1
    return t


def reset_outputs(b, stream=None):
    """stats = 0, status = -1 with one device-to-device copy (the step's only reset op)."""
    b.in_arena[b.in_arena.numel() - b.reset.numel():].copy_(b.reset, non_blocking=True)


def make_batch(profiles_gain: List[np.ndarray], profiles_cost: List[np.ndarray], profiles_shape: List[tuple],
               num_frames: np.ndarray, budget_bound: np.ndarray, profile: np.ndarray,
               class_id: Optional[np.ndarray] = None, capacity: Optional[np.ndarray] = None,
               base_cost: int = 0, device="cuda", with_plan_workspace: bool = True) -> Batch:
    """Allocate device buffers for a batch and size it (turbo_mckp_workspace).

    budget_bound: per-window budget used for the layout (the true budget, or an upper
    bound when a1 derives the budget on device from capacity)."""
    import torch
    load()
    dev = torch.device(device)
    ptens, phost = [], []
    for g, c, (C, K) in zip(profiles_gain, profiles_cost, profiles_shape):
        gt = torch.as_tensor(np.ascontiguousarray(g, dtype=np.int32), device=dev)
        ct = torch.as_tensor(np.ascontiguousarray(c, dtype=np.int32), device=dev)
        ptens += [gt, ct]
        phost.append(Profile(int(C), int(K), gt.data_ptr(), ct.data_ptr()))
    W = len(num_frames)
    wins = np.zeros(W, dtype=WINDOW_DTYPE)
    nf = np.asarray(num_frames, dtype=np.int64)
    ff = np.zeros(W, dtype=np.int64)
    if W > 1:
        ff[1:] = np.cumsum(nf[:-1])
    wins["first_frame"] = ff
    wins["num_frames"] = nf
    wins["budget"] = np.asarray(budget_bound, dtype=np.int32)
    wins["profile"] = np.asarray(profile, dtype=np.int32)
    shape = mckp_workspace(phost, wins)
    pbytes = np.frombuffer(bytes((Profile * max(len(phost), 1))(*phost)), dtype=np.uint8)
    profiles_dev = torch.as_tensor(pbytes.copy(), device=dev)
    windows_dev = torch.as_tensor(wins.view(np.uint8).copy(), device=dev)
    F = int(shape.total_frames)
    # One device arena, 16-B aligned sections:
    #   [capacity int32 W | class_id u8 F | stats int64 181 | status int64 2 |
    #    best_gain int32 W | best_cost int32 W | feasible u8 W | exit_out u8 F]
    # in_arena = the first four sections (ONE host->device copy per step carries the inputs AND the
    # initial stats (0) / status (-1)); out_arena = stats .. exit_out (ONE device->host copy).
    def _carve(arena, sizes):
        views, off, offs = [], 0, []
        for nbytes, dt in sizes:
            views.append(arena[off: off + nbytes].view(dt))
            offs.append(off)
            off += (nbytes + 15) & ~15
        return views, offs, off
    sizes = [(4 * max(W, 1), torch.int32), (max(F, 1), torch.uint8), (8 * STATS_WORDS, torch.int64),
             (8 * STATUS_WORDS, torch.int64), (4 * max(W, 1), torch.int32), (4 * max(W, 1), torch.int32),
             (max(W, 1), torch.uint8), (max(F, 1), torch.uint8)]
    total = sum((n + 15) & ~15 for n, _ in sizes)
    arena = torch.zeros(total, dtype=torch.uint8, device=dev)
    (cap_v, cls, st_v, status_v, bg_v, bc_v, fe_v, ex_v), offs, _ = _carve(arena, sizes)
    in_arena = arena[: offs[4]]
    out_arena = arena[offs[2]:]
    if class_id is not None and F:
        cls[:F] = torch.as_tensor(np.ascontiguousarray(class_id, dtype=np.uint8), device=dev)
    cap = None
    if capacity is not None:
        cap = cap_v
        cap[:W] = torch.as_tensor(np.ascontiguousarray(capacity, dtype=np.int32), device=dev)
    status_v.fill_(-1)
    nopt = max(int(shape.total_options), 4)
    ws_bytes = int(shape.workspace_bytes) if with_plan_workspace else 0
    solve_bytes = mckp_solve_workspace(shape)
    return Batch(shape=shape, windows_host=wins, profiles_host=phost, profile_tensors=ptens,
                 profiles_dev=profiles_dev, windows_dev=windows_dev, class_id=cls, capacity=cap,
                 base_cost=int(base_cost),
                 opt_gain=torch.zeros(nopt, dtype=torch.int32, device=dev),
                 opt_cost=torch.zeros(nopt, dtype=torch.int32, device=dev),
                 workspace=torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev) if ws_bytes else None,
                 best_gain=bg_v, best_cost=bc_v, feasible=fe_v, exit_out=ex_v, status=status_v, stats=st_v,
                 solve_ws=torch.empty(solve_bytes, dtype=torch.uint8, device=dev) if solve_bytes else None,
                 in_arena=in_arena, out_arena=out_arena, reset=_reset_template(arena, offs))


def batch_from_workload(wl, device="cuda", with_plan_workspace: bool = True, null_capacity: bool = False) -> Batch:
    """Device batch for a synth.Workload (budgets derived on device by a1 from capacity; with
    null_capacity the calls get capacity = NULL and plan the windows' own budget fields)."""
    return make_batch(wl.profiles_gain, wl.profiles_cost, wl.profiles_shape, wl.num_frames, wl.budget,
                      wl.profile, wl.class_id, None if null_capacity else wl.capacity, wl.base_cost, device,
                      with_plan_workspace)


def set_device_budgets(b: Batch, budgets: np.ndarray):
    """Overwrite turbo_window_t.budget of the DEVICE window array (the layout bound stays as sized):
    what a caller does when it derives budgets itself and passes capacity = NULL."""
    import torch
    wins = b.windows_dev.cpu().numpy().view(WINDOW_DTYPE).copy()
    wins["budget"] = np.asarray(budgets, dtype=np.int32)
    b.windows_dev.copy_(torch.as_tensor(wins.view(np.uint8)))


def run_path(b: Batch, fused=True, stream=None, with_stats: bool = True, reset: bool = True):
    """One pass of the hot path: a1+a2 lookup -> a3..a5 (solve, or plan + backtrack) -> a6 stats.
    fused="all" runs the single-launch turbo_schedule (a1..a6) instead."""
    if reset:
        b.status.fill_(-1)
        if with_stats:
            b.stats.zero_()
    if fused == "all":
        schedule(b.shape, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost, b.solve_ws,
                 b.best_gain, b.best_cost, b.feasible, b.exit_out, b.stats, b.status, stream)
        return
    profile_lookup(b.shape, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost, b.opt_gain,
                   b.opt_cost, b.status, stream)
    if fused:
        mckp_solve(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, b.solve_ws, b.best_gain, b.best_cost,
                   b.feasible, b.exit_out, b.status, stream)
    else:
        mckp_plan(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, b.workspace, b.best_gain, b.best_cost,
                  b.feasible, b.status, stream)
        backtrack(b.shape, b.windows_dev, b.opt_cost, b.workspace, b.best_cost, b.feasible, b.exit_out, stream)
    if with_stats:
        stats(b.shape, b.windows_dev, b.class_id, b.exit_out, b.best_gain, b.best_cost, b.feasible, b.stats,
              stream)


def results(b: Batch) -> dict:
    """Copy the outputs back to the host (numpy)."""
    W = int(b.shape.num_windows)
    F = int(b.shape.total_frames)
    wins = b.windows_dev.cpu().numpy().view(WINDOW_DTYPE)
    return dict(exits=b.exit_out[:F].cpu().numpy(), best_gain=b.best_gain[:W].cpu().numpy(),
                best_cost=b.best_cost[:W].cpu().numpy(), feasible=b.feasible[:W].cpu().numpy(),
                status=b.status.cpu().numpy(), stats=b.stats.cpu().numpy(), budget=wins["budget"].copy(),
                opt_gain=b.opt_gain.cpu().numpy(), opt_cost=b.opt_cost.cpu().numpy(),
                first_option=b.windows_host["first_option"].copy())

"""CPU oracle for the Turbo MCKP scheduler hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package. The product package paper_2207_00172_b200 never
imports it and shares no code with it (see oracle/turbo_oracle.c header).

Functions follow /root/reference/PAPER.md §5 (lines 491-545) and §6.4 (line 858);
see turbo_oracle.c for the per-function citations and DESIGN.md for readings.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "turbo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-pthread",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def profiles_flat(wl):
    """Concatenate profile tables: (gain, cost, offset[P], C[P], K[P])."""
    gain = np.concatenate([_i32(g) for g in wl.profiles_gain]) if wl.profiles_gain else np.zeros(0, np.int32)
    cost = np.concatenate([_i32(c) for c in wl.profiles_cost]) if wl.profiles_cost else np.zeros(0, np.int32)
    sizes = np.array([len(g) for g in wl.profiles_gain], dtype=np.int64)
    off = np.zeros(len(sizes), dtype=np.int64)
    if len(sizes) > 1:
        off[1:] = np.cumsum(sizes[:-1])
    C = np.array([s[0] for s in wl.profiles_shape], dtype=np.int32)
    K = np.array([s[1] for s in wl.profiles_shape], dtype=np.int32)
    return _i32(gain), _i32(cost), off, C, K


def option_offsets(num_frames, K):
    """first_option[w] = sum_{w' < w} N_w' K_w' (layout bookkeeping only)."""
    n = np.asarray(num_frames, dtype=np.int64) * np.asarray(K, dtype=np.int64)
    off = np.zeros(len(n), dtype=np.int64)
    if len(n) > 1:
        off[1:] = np.cumsum(n[:-1])
    return off, int(n.sum())


def budget(capacity, num_frames, base_cost) -> np.ndarray:
    lib = _load()
    cap, nf = _i32(capacity), _i32(num_frames)
    out = np.zeros(len(nf), dtype=np.int32)
    lib.oracle_budget(ctypes.c_int32(len(nf)), _p(cap), _p(nf), ctypes.c_int32(int(base_cost)), _p(out))
    return out


def lookup(wl):
    """a2: per-frame option tables. Returns (opt_gain, opt_cost, first_option, bad_frame)."""
    lib = _load()
    gain, cost, off, C, K = profiles_flat(wl)
    Kw = K[wl.profile]
    first_option, total = option_offsets(wl.num_frames, Kw)
    og = np.zeros(max(total, 1), dtype=np.int32)
    oc = np.zeros(max(total, 1), dtype=np.int32)
    cls = np.ascontiguousarray(wl.class_id, dtype=np.uint8)
    lib.oracle_lookup.restype = ctypes.c_int64
    bad = lib.oracle_lookup(ctypes.c_int32(wl.num_windows), _p(_i32(wl.num_frames)), _p(_i32(wl.profile)),
                            _p(cls), _p(gain), _p(cost), _p(off), _p(C), _p(K), _p(og), _p(oc))
    return og[:total], oc[:total], first_option, int(bad)


def plan(num_frames, budget_, K, opt_gain, opt_cost, mode: str = "table",
         threads: Optional[int] = None):
    """a3-a5 per window. mode: 'table' | 'brute' | 'value' (no exits)."""
    lib = _load()
    nf, bud, Kw = _i32(num_frames), _i32(budget_), _i32(K)
    W = len(nf)
    ff = np.zeros(W, dtype=np.int64)
    if W > 1:
        ff[1:] = np.cumsum(nf[:-1].astype(np.int64))
    fo, total = option_offsets(nf, Kw)
    F = int(nf.astype(np.int64).sum())
    exits = np.zeros(max(F, 1), dtype=np.uint8)
    bg = np.zeros(max(W, 1), dtype=np.int64)
    bc = np.zeros(max(W, 1), dtype=np.int64)
    fe = np.zeros(max(W, 1), dtype=np.uint8)
    og = _i32(opt_gain) if total else np.zeros(1, np.int32)
    oc = _i32(opt_cost) if total else np.zeros(1, np.int32)
    m = {"table": 0, "brute": 1, "value": 2}[mode]
    nt = threads or min(os.cpu_count() or 1, 64)
    err = lib.oracle_plan_batch(ctypes.c_int32(W), _p(nf), _p(bud), _p(Kw), _p(ff), _p(fo), _p(og), _p(oc),
                                _p(exits), _p(bg), _p(bc), _p(fe), ctypes.c_int32(m), ctypes.c_int32(nt))
    if err:
        raise RuntimeError(f"oracle_plan_batch failed: {err}")
    return exits[:F], bg[:W], bc[:W], fe[:W]


def heuristic(num_frames, budget_, K, opt_gain, opt_cost):
    """NEXT-1: the paper's prune-and-search heuristic per window.
    Returns (exits, gain, cost, feasible, steps)."""
    lib = _load()
    nf, bud, Kw = _i32(num_frames), _i32(budget_), _i32(K)
    W = len(nf)
    ff = np.zeros(W, dtype=np.int64)
    if W > 1:
        ff[1:] = np.cumsum(nf[:-1].astype(np.int64))
    fo, total = option_offsets(nf, Kw)
    F = int(nf.astype(np.int64).sum())
    exits = np.zeros(max(F, 1), dtype=np.uint8)
    g = np.zeros(max(W, 1), dtype=np.int64)
    c = np.zeros(max(W, 1), dtype=np.int64)
    fe = np.zeros(max(W, 1), dtype=np.uint8)
    st = np.zeros(max(W, 1), dtype=np.int64)
    og = _i32(opt_gain) if total else np.zeros(1, np.int32)
    oc = _i32(opt_cost) if total else np.zeros(1, np.int32)
    lib.oracle_heuristic_batch(ctypes.c_int32(W), _p(nf), _p(bud), _p(Kw), _p(ff), _p(fo), _p(og), _p(oc),
                               _p(exits), _p(g), _p(c), _p(fe), _p(st))
    return exits[:F], g[:W], c[:W], fe[:W], st[:W]


def bucketize(theta, num_classes: int = 10, width: float = 0.1) -> np.ndarray:
    """NEXT-3: class = clamp(floor((1 - theta) * (1/width)), 0, C-1) in float32."""
    lib = _load()
    th = np.ascontiguousarray(theta, dtype=np.float32)
    out = np.zeros(max(len(th), 1), dtype=np.uint8)
    lib.oracle_bucketize(ctypes.c_int64(len(th)), _p(th), ctypes.c_float(np.float32(1.0) / np.float32(width)),
                         ctypes.c_int32(num_classes), _p(out))
    return out[:len(th)]


def batches(num_frames, exits):
    """NEXT-2: per-window exit counts [W, 16] and the stable per-exit frame order [F]."""
    lib = _load()
    nf = _i32(num_frames)
    W = len(nf)
    F = int(nf.astype(np.int64).sum())
    count = np.zeros(max(W, 1) * 16, dtype=np.int32)
    order = np.zeros(max(F, 1), dtype=np.int32)
    lib.oracle_batches(ctypes.c_int32(W), _p(nf), _p(np.ascontiguousarray(exits, dtype=np.uint8)), _p(count),
                       _p(order))
    return count[:W * 16].reshape(W, 16), order[:F]


def batch_latency(count16, num_exits, profile, profiles_batch, ncap: int) -> np.ndarray:
    """NEXT-2 executed latency per window: sum_k I_k(n_k) over the window's levels;
    profiles_batch[p] = int32 [K_p * (ncap + 1)] (row k = I_k(0..ncap)); -1 when some n_k > ncap."""
    lib = _load()
    cnt = np.ascontiguousarray(count16, dtype=np.int32).reshape(-1)
    W = len(cnt) // 16
    tabs = np.concatenate([_i32(t) for t in profiles_batch])
    sz = np.array([len(t) for t in profiles_batch], dtype=np.int64)
    off = np.zeros(len(sz), dtype=np.int64)
    off[1:] = np.cumsum(sz[:-1])
    out = np.zeros(max(W, 1), dtype=np.int64)
    lib.oracle_batch_latency(ctypes.c_int32(W), _p(cnt), _p(_i32(num_exits)), _p(tabs), _p(off), _p(_i32(profile)),
                             ctypes.c_int32(int(ncap)), _p(out))
    return out[:W]


def stats(num_frames, class_id, exits, best_gain, best_cost, feasible) -> np.ndarray:
    lib = _load()
    out = np.zeros(181, dtype=np.int64)
    nf = _i32(num_frames)
    lib.oracle_stats(ctypes.c_int32(len(nf)), _p(nf), _p(np.ascontiguousarray(class_id, dtype=np.uint8)),
                     _p(np.ascontiguousarray(exits, dtype=np.uint8)), _p(_i64(best_gain)), _p(_i64(best_cost)),
                     _p(np.ascontiguousarray(feasible, dtype=np.uint8)), _p(out))
    return out


def run(wl, mode: str = "table", threads: Optional[int] = None, budgets=None) -> dict:
    """The whole path a1..a6 on one workload (budgets given: the capacity = NULL path, a1 skipped)."""
    bud = budget(wl.capacity, wl.num_frames, wl.base_cost) if budgets is None else _i32(budgets)
    og, oc, fo, bad = lookup(wl)
    K = wl.num_exits
    exits, bg, bc, fe = plan(wl.num_frames, bud, K, og, oc, mode, threads)
    st = stats(wl.num_frames, wl.class_id, exits, bg, bc, fe) if mode != "value" else None
    return dict(budget=bud, opt_gain=og, opt_cost=oc, first_option=fo, bad_frame=bad,
                exits=exits, best_gain=bg, best_cost=bc, feasible=fe, stats=st)


def batched_brute(cls, gain, C, K, batch, ncap, B):
    """NEXT-4, one tiny window by enumeration of all K^N plans (turbo_oracle.c
    oracle_batched_brute). Returns (G*, C*, counts of the lexicographically smallest optimal
    count vector, feasible)."""
    lib = _load()
    cl = np.ascontiguousarray(cls, dtype=np.uint8)
    g, I = _i32(gain), _i32(batch)
    bg, bc = ctypes.c_int64(0), ctypes.c_int64(0)
    cnt = np.zeros(16, dtype=np.int32)
    fe = ctypes.c_uint8(0)
    e = lib.oracle_batched_brute(ctypes.c_int32(len(cl)), ctypes.c_int32(C), ctypes.c_int32(K), _p(cl), _p(g), _p(I),
                                 ctypes.c_int32(ncap), ctypes.c_int32(int(B)), ctypes.byref(bg), ctypes.byref(bc),
                                 _p(cnt), ctypes.byref(fe))
    if e:
        raise RuntimeError(f"oracle_batched_brute failed: {e}")
    return int(bg.value), int(bc.value), cnt[:K].copy(), int(fe.value)


def _batched_one(fn, cls, gain, C, K, batch, ncap, B):
    lib = _load()
    cl = np.ascontiguousarray(cls, dtype=np.uint8)
    ex = np.zeros(max(len(cl), 1), dtype=np.uint8)
    bg, bc = ctypes.c_int64(0), ctypes.c_int64(0)
    fe = ctypes.c_uint8(0)
    e = getattr(lib, fn)(ctypes.c_int32(len(cl)), ctypes.c_int32(C), ctypes.c_int32(K), _p(cl), _p(_i32(gain)),
                         _p(_i32(batch)), ctypes.c_int32(ncap), ctypes.c_int32(int(B)), _p(ex), ctypes.byref(bg),
                         ctypes.byref(bc), ctypes.byref(fe))
    if e:
        raise RuntimeError(f"{fn} failed: {e}")
    return ex[:len(cl)].copy(), int(bg.value), int(bc.value), int(fe.value)


def batched_dp(cls, gain, C, K, batch, ncap, B):
    """NEXT-4 for any gain table (reading R20), one window: the DP over the canonical prefix and its
    count vector (turbo_oracle.c oracle_batched_dp). Returns (exits, G*, C*, feasible)."""
    return _batched_one("oracle_batched_dp", cls, gain, C, K, batch, ncap, B)


def batched_brute_plan(cls, gain, C, K, batch, ncap, B):
    """The R20 plan by its definition over all K^N plans (N <= 12). Returns (exits, G*, C*, feasible)."""
    return _batched_one("oracle_batched_brute_plan", cls, gain, C, K, batch, ncap, B)


def batched_enum(cls, gain, C, K, batch, ncap, B):
    """NEXT-4 under R19 (count vectors + canonical assignment), one window; raises on an R19 violation."""
    return _batched_one("oracle_batched_enum", cls, gain, C, K, batch, ncap, B)


def batched(wl):
    """NEXT-4 on a batched workload (synth profiles_batch): exact optimum per window by
    count-vector enumeration (turbo_oracle.c oracle_batched_enum) when the gains satisfy R19, else
    by the general program (oracle_batched_dp, reading R20). Returns (exits, G*, C*, feasible)."""
    lib = _load()
    gain = np.concatenate([_i32(g) for g in wl.profiles_gain])
    gsz = np.array([len(g) for g in wl.profiles_gain], dtype=np.int64)
    goff = np.zeros(len(gsz), dtype=np.int64)
    goff[1:] = np.cumsum(gsz[:-1])
    bt = np.concatenate([_i32(t) for t in wl.profiles_batch])
    bsz = np.array([len(t) for t in wl.profiles_batch], dtype=np.int64)
    boff = np.zeros(len(bsz), dtype=np.int64)
    boff[1:] = np.cumsum(bsz[:-1])
    C = np.array([s[0] for s in wl.profiles_shape], dtype=np.int32)
    K = np.array([s[1] for s in wl.profiles_shape], dtype=np.int32)
    W = wl.num_windows
    F = wl.total_frames
    ff = _i64(wl.first_frame)
    exits = np.zeros(max(F, 1), dtype=np.uint8)
    bg = np.zeros(max(W, 1), dtype=np.int64)
    bc = np.zeros(max(W, 1), dtype=np.int64)
    fe = np.zeros(max(W, 1), dtype=np.uint8)
    cls = np.ascontiguousarray(wl.class_id, dtype=np.uint8)
    e = lib.oracle_batched_batch(ctypes.c_int32(W), _p(_i32(wl.num_frames)), _p(_i32(wl.budget)), _p(_i32(wl.profile)),
                                 _p(ff), _p(cls if F else np.zeros(1, np.uint8)), _p(gain), _p(goff), _p(C), _p(K),
                                 _p(bt), _p(boff), ctypes.c_int32(wl.batch_cap), _p(exits), _p(bg), _p(bc), _p(fe))
    if e:
        raise RuntimeError(f"oracle_batched_batch failed: {e}")
    return exits[:F], bg[:W], bc[:W], fe[:W]

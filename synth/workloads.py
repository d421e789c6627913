"""Named synthetic workloads (BASELINE.json configs c1..c5) plus parity-only sets.

Every array here is an INPUT of the hot path. Nothing in this file evaluates the
scheduler (no budget rule, no lookup, no knapsack): `capacity` is produced as
budget + N * base_cost so that the a1 budget rule, applied by the code under
test, must give back the configured budget (reading R3).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .rng import rand_int, rand_uniform

NUM_CLASSES = 10                 # buckets of width 0.1
BASE_SEED = 220700172            # seed_k = BASE_SEED + k

# stream ids (one per independent random quantity)
S_CLASS, S_LAMBDA, S_BURST, S_BURSTC, S_BURSTU = 1, 2, 3, 4, 5
S_K, S_B, S_N, S_PROF, S_TGAIN, S_TCOST, S_TBASE, S_TBUD, S_TN = range(6, 15)


@dataclass
class Workload:
    """A batch of scheduling windows and the offline profiles they reference."""
    name: str
    profiles_gain: List[np.ndarray]          # per profile: int32 [C*K], row-major (class, exit)
    profiles_cost: List[np.ndarray]          # per profile: int32 [C*K]
    profiles_shape: List[tuple]              # per profile: (C, K)
    num_frames: np.ndarray                   # int32 [W]  m_w
    budget: np.ndarray                       # int32 [W]  B_w (config value; = a1 result)
    capacity: np.ndarray                     # int32 [W]  floor(T_w/q) (input of a1)
    base_cost: int                           # u0 = ceil(I_0/q) (input of a1)
    profile: np.ndarray                      # int32 [W]  profile index per window
    class_id: np.ndarray                     # uint8 [F]  concatenated per window
    meta: dict = field(default_factory=dict)
    # NEXT-4 (batched cost): per profile int32 [K * (batch_cap + 1)], I_k(n) = latency of a batch
    # of n frames at level k (row-major (level, n)); None for the per-frame-cost workloads
    profiles_batch: Optional[List[np.ndarray]] = None
    batch_cap: int = 0

    @property
    def num_windows(self) -> int:
        return int(self.num_frames.shape[0])

    @property
    def first_frame(self) -> np.ndarray:
        ff = np.zeros(self.num_windows, dtype=np.int64)
        if self.num_windows > 1:
            ff[1:] = np.cumsum(self.num_frames[:-1].astype(np.int64))
        return ff

    @property
    def num_exits(self) -> np.ndarray:
        ks = np.array([s[1] for s in self.profiles_shape], dtype=np.int32)
        return ks[self.profile]

    @property
    def total_frames(self) -> int:
        return int(self.num_frames.astype(np.int64).sum())

    @property
    def total_cells(self) -> int:
        """Sum over windows of N_w (B_w + 1): the cell-updates of one DP pass."""
        return int((self.num_frames.astype(np.int64) * (self.budget.astype(np.int64) + 1)).sum())

    def subset(self, lo: int, hi: int, name: Optional[str] = None) -> "Workload":
        """Contiguous window range [lo, hi) sharing the same profiles."""
        ff = self.first_frame
        f0 = int(ff[lo]) if lo < self.num_windows else self.total_frames
        f1 = int(ff[hi]) if hi < self.num_windows else self.total_frames
        return Workload(name or f"{self.name}[{lo}:{hi}]", self.profiles_gain, self.profiles_cost,
                        self.profiles_shape, self.num_frames[lo:hi].copy(), self.budget[lo:hi].copy(),
                        self.capacity[lo:hi].copy(), self.base_cost, self.profile[lo:hi].copy(),
                        self.class_id[f0:f1].copy(), dict(self.meta))


# ----------------------------------------------------------------------------- profiles
def paper_gain_table(K: int, C: int = NUM_CLASSES) -> np.ndarray:
    """Appendix-B calibrated accuracy profile P_k^theta in 0.01 mAP points (int32 [C*K])."""
    g = np.zeros((C, K), dtype=np.int64)
    for c in range(C):
        amp = 1400.0 * 0.604 ** (9 - c)
        for k in range(1, K):
            frac = 1.0 if K == 2 else 0.561 + 0.439 * (k - 1) / (K - 2)
            g[c, k] = int(math.floor(amp * frac + 0.5))
    return g.reshape(-1).astype(np.int32)


def regular_costs(K: int, c_max: int) -> np.ndarray:
    """c_k = ceil(c_max k / (K-1)) (integer ceil), k = 0..K-1."""
    return np.array([-((-c_max * k) // (K - 1)) for k in range(K)], dtype=np.int64)


def _paper_profile(K: int, c_max: int, C: int = NUM_CLASSES):
    gain = paper_gain_table(K, C)
    cost = np.tile(regular_costs(K, c_max), C).astype(np.int32)
    return gain, cost


def _class_ids(seed: int, num_frames: np.ndarray, lam: np.ndarray,
               burst: Optional[np.ndarray] = None, burst_class: Optional[np.ndarray] = None,
               window_ids: Optional[np.ndarray] = None) -> np.ndarray:
    """Per-frame classes: P(c) ∝ exp(-lam_w c); burst windows put ~85% of frames on one class."""
    W = num_frames.shape[0]
    wid = np.arange(W, dtype=np.int64) if window_ids is None else window_ids.astype(np.int64)
    nf = num_frames.astype(np.int64)
    F = int(nf.sum())
    if F == 0:
        return np.zeros(0, dtype=np.uint8)
    w_of = np.repeat(np.arange(W), nf)
    first = np.zeros(W, dtype=np.int64)
    first[1:] = np.cumsum(nf[:-1])
    j = np.arange(F, dtype=np.int64) - first[w_of]
    u = rand_uniform(seed, S_CLASS * 2**40 + wid[w_of], j)
    cs = np.arange(NUM_CLASSES, dtype=np.float64)
    # per-window cdf (lam may differ per window)
    lam_w = np.broadcast_to(np.asarray(lam, dtype=np.float64), (W,))
    pw = np.exp(-lam_w[:, None] * cs[None, :])
    cdf = np.cumsum(pw, axis=1)
    cdf /= cdf[:, -1:]
    cls = (u[:, None] >= cdf[w_of]).sum(axis=1)
    cls = np.minimum(cls, NUM_CLASSES - 1)
    if burst is not None:
        ub = rand_uniform(seed, S_BURSTU * 2**40 + wid[w_of], j)
        take = burst[w_of] & (ub < 0.85)
        cls = np.where(take, burst_class[w_of], cls)
    return cls.astype(np.uint8)


def _wl(name, gains, costs, shapes, nf, bud, prof, cls, base_cost, meta=None):
    nf = np.asarray(nf, dtype=np.int32)
    bud = np.asarray(bud, dtype=np.int32)
    cap = (bud.astype(np.int64) + nf.astype(np.int64) * base_cost).astype(np.int32)
    return Workload(name, gains, costs, shapes, nf, bud, cap, int(base_cost),
                    np.asarray(prof, dtype=np.int32), np.asarray(cls, dtype=np.uint8), meta or {})


# ----------------------------------------------------------------------------- configs
def _uniform_config(k: int, W: int, N: int, K: int, B: int, window_offset: int = 0,
                    num_windows: Optional[int] = None, base_cost: int = 84) -> Workload:
    seed = BASE_SEED + k
    c_max = -((-3 * B) // N)
    g, c = _paper_profile(K, c_max)
    Wl = W if num_windows is None else num_windows
    wid = np.arange(window_offset, window_offset + Wl, dtype=np.int64)
    nf = np.full(Wl, N, dtype=np.int32)
    cls = _class_ids(seed, nf, np.full(Wl, 0.35), window_ids=wid)
    return _wl(f"c{k}", [g], [c], [(NUM_CLASSES, K)], nf, np.full(Wl, B), np.zeros(Wl), cls,
               base_cost, {"config": k, "N": N, "K": K, "B": B, "W_total": W,
                           "window_offset": window_offset, "c_max": c_max})


def _c5(W: int = 16384, window_offset: int = 0, num_windows: Optional[int] = None) -> Workload:
    """Mixed sweep: K ~ U{2..16}, B = round(64 * 256**u), N = 30 U{1..10}, skewed histograms."""
    seed = BASE_SEED + 5
    Wl = W if num_windows is None else num_windows
    wid = np.arange(window_offset, window_offset + Wl, dtype=np.int64)
    K = rand_int(seed, S_K, wid, 2, 16)
    u = rand_uniform(seed, S_B, wid)
    B = np.floor(64.0 * 256.0 ** u + 0.5).astype(np.int64)
    N = 30 * rand_int(seed, S_N, wid, 1, 10)
    lam = -0.5 + 2.0 * rand_uniform(seed, S_LAMBDA, wid)
    burst = rand_uniform(seed, S_BURST, wid) < 0.05
    bcls = rand_int(seed, S_BURSTC, wid, 0, NUM_CLASSES - 1)
    # profiles: one per (K, cost scale s), c_max = 2**s with s = ceil(log2(ceil(3B/N)))
    cm = -((-3 * B) // N)
    s = np.ceil(np.log2(np.maximum(cm, 1))).astype(np.int64)
    s = np.clip(s, 0, 11)
    prof = (K - 2) * 12 + s
    gains, costs, shapes = [], [], []
    for kk in range(2, 17):
        for ss in range(12):
            g, c = _paper_profile(kk, 2 ** ss)
            gains.append(g)
            costs.append(c)
            shapes.append((NUM_CLASSES, kk))
    cls = _class_ids(seed, N, lam, burst, bcls, window_ids=wid)
    return _wl("c5", gains, costs, shapes, N, B, prof, cls, 84,
               {"config": 5, "W_total": W, "window_offset": window_offset})


CONFIGS = {
    1: dict(W=1, N=30, K=4, B=120),
    2: dict(W=1024, N=30, K=5, B=1000),
    3: dict(W=65536, N=300, K=8, B=4096),
    4: dict(W=1, N=3000, K=6, B=1 << 20),
}


def make_config(k: int, window_offset: int = 0, num_windows: Optional[int] = None) -> Workload:
    """Config k of BASELINE.json (1..5); optionally only windows [offset, offset+num)."""
    if k == 5:
        return _c5(window_offset=window_offset, num_windows=num_windows)
    p = CONFIGS[k]
    return _uniform_config(k, p["W"], p["N"], p["K"], p["B"], window_offset, num_windows)


# ----------------------------------------------------------------------------- parity sets
def make_tie_heavy(seed: int, W: int, max_frames: int = 8, max_exits: int = 4,
                   num_profiles: int = 16, max_budget: Optional[int] = None,
                   C: int = NUM_CLASSES, base_cost: int = 3, fixed_exits: Optional[int] = None,
                   max_cost: int = 4) -> Workload:
    """Gains U{-2..8}, costs U{0..max_cost}; 30% of profiles have c_0 > 0 (infeasible windows).
    fixed_exits: every profile has that K (else K ~ U{2..max_exits} per profile)."""
    gains, costs, shapes = [], [], []
    for p in range(num_profiles):
        K = int(rand_int(seed, S_PROF, p, 2, max_exits)) if fixed_exits is None else int(fixed_exits)
        n = C * K
        g = rand_int(seed, S_TGAIN, p * 4096 + np.arange(n), -2, 8).astype(np.int32)
        c = rand_int(seed, S_TCOST, p * 4096 + np.arange(n), 0, max_cost).astype(np.int32)
        if rand_uniform(seed, S_TBASE, p) >= 0.3:
            c.reshape(C, K)[:, 0] = 0
        gains.append(g)
        costs.append(c)
        shapes.append((C, K))
    wid = np.arange(W)
    N = rand_int(seed, S_TN, wid, 0, max_frames).astype(np.int32)
    hi = 3 * np.maximum(N, 1) if max_budget is None else np.full(W, max_budget)
    B = rand_int(seed, S_TBUD, wid, 0, hi).astype(np.int32)
    prof = rand_int(seed, S_PROF + 100, wid, 0, num_profiles - 1).astype(np.int32)
    u = rand_uniform(seed, S_CLASS, np.arange(int(N.sum())))
    cls = np.minimum((u * C).astype(np.int64), C - 1)
    return _wl(f"tie{seed}", gains, costs, shapes, N, B, prof, cls, base_cost, {"seed": seed})


def make_adversarial() -> Workload:
    """SURVEY.md §8(c) adversarial parity set, one window per case (C = 1 profiles).

    Each profile is a single class row; windows list their frames' option rows by
    giving every frame its own profile class. Cases 1..15 of SURVEY.md §8(c)."""
    cases = []  # (list of per-frame rows [(g, c), ...], budget)

    def rows(*r):
        return [list(x) for x in r]

    cases.append(([], 5))                                                   # 1: N = 0
    cases.append((rows([(0, 0), (3, 1)], [(0, 0), (2, 2)]), 0))            # 2: B = 0
    cases.append((rows([(0, 0), (5, 7)], [(0, 0), (4, 9)]), 6))            # 3: B < all non-zero c
    cases.append((rows([(0, 0), (5, 0), (7, 0)], [(1, 0), (2, 0), (2, 0)]), 0))    # 4: all costs 0
    cases.append((rows([(0, 0), (9, 50)], [(0, 0), (9, 51)]), 49))         # 5: c > B for k >= 1
    cases.append((rows(*[[(0, 0), (k % 3, 1)] for k in range(7)]), 4))      # 6a: K = 2
    cases.append((rows(*[[(k * j % 11, j) for j in range(16)] for k in range(5)]), 37))  # 6b: K = 16
    cases.append((rows(*[[(5, 0), (5, 1), (5, 2)] for _ in range(6)]), 7))  # 7: all-equal gains
    cases.append((rows([(0, 0), (3, 2)], [(0, 0), (3, 5)]), 5))            # 8: cost-before-lex
    cases.append((rows([(0, 0), (4, 5)], [(0, 0), (4, 5)]), 5))            # 9: lex
    cases.append((rows([(0, 0), (4, 5), (4, 7)]), 10))                     # 10: min cost in frame
    cases.append((rows([(-3, 0), (-1, 2)], [(-5, 0), (-6, 1)], [(0, 0), (-2, 3)]), 4))  # 11: negative
    cases.append((rows([(2, 3), (5, 6)], [(1, 2), (9, 9)]), 4))            # 12: c_0 > 0 infeasible
    cases.append((rows(*[[(0, 0), (7, 33), (9, 257), (11, 300)] for _ in range(5)]), 700))  # 13: chunk-crossing
    cases.append((rows(*[[(0, 0), (3, 31), (8, 95)] for _ in range(4)]), 288))  # 14: B+1 not mult of 32
    big = 32767
    cases.append((rows(*[[(0, 0), (big, 1), (-big, 0)] for _ in range(1000)]), 999))  # 15: range limit
    # one profile per distinct frame row keeps C small; K = max len, short rows padded by copies
    # of an infeasible option is NOT allowed (changes semantics) -> group windows by K instead.
    gains, costs, shapes = [], [], []
    nf, bud, prof, cls = [], [], [], []
    for frames, B in cases:
        K = max((len(r) for r in frames), default=2)
        uniq = []
        for r in frames:
            assert len(r) == K
            if r not in uniq:
                uniq.append(r)
        C = max(len(uniq), 1)
        g = np.zeros((C, K), dtype=np.int32)
        c = np.zeros((C, K), dtype=np.int32)
        for x, r in enumerate(uniq):
            for k, (gg, cc) in enumerate(r):
                g[x, k], c[x, k] = gg, cc
        gains.append(g.reshape(-1))
        costs.append(c.reshape(-1))
        shapes.append((C, K))
        nf.append(len(frames))
        bud.append(B)
        prof.append(len(gains) - 1)
        cls.extend(uniq.index(r) for r in frames)
    return _wl("adversarial", gains, costs, shapes, nf, bud, prof, cls, 2)


def concat_workloads(parts: List[Workload], name: str = "concat") -> Workload:
    """Concatenate windows of several workloads (profiles are re-indexed)."""
    gains, costs, shapes, nf, bud, cap, prof, cls = [], [], [], [], [], [], [], []
    base = parts[0].base_cost
    for p in parts:
        assert p.base_cost == base
        off = len(gains)
        gains += p.profiles_gain
        costs += p.profiles_cost
        shapes += p.profiles_shape
        nf.append(p.num_frames)
        bud.append(p.budget)
        cap.append(p.capacity)
        prof.append(p.profile + off)
        cls.append(p.class_id)
    return Workload(name, gains, costs, shapes, np.concatenate(nf), np.concatenate(bud),
                    np.concatenate(cap), base, np.concatenate(prof), np.concatenate(cls), {})


def make_long_window(seed: int, N: int, K: int, B: int, c_max: Optional[int] = None, random_rows: bool = False,
                     C: int = NUM_CLASSES, base_cost: int = 84) -> Workload:
    """One long window (c4-shaped: rows far beyond one CTA). Paper profile with regular costs
    c_max = ceil(3B/N), or (random_rows) gains U{-2..40}, costs U{0..c_max}, c_0 = 0."""
    cm = -((-3 * B) // N) if c_max is None else c_max
    if random_rows:
        g = rand_int(seed, S_TGAIN, np.arange(C * K), -2, 40).astype(np.int32)
        c = rand_int(seed, S_TCOST, np.arange(C * K), 0, cm).astype(np.int32)
        c.reshape(C, K)[:, 0] = 0
    else:
        g, c = _paper_profile(K, cm, C)
    cls = _class_ids(seed, np.array([N], np.int32), np.array([0.35]), window_ids=np.array([seed]))
    return _wl(f"long{seed}", [g], [c], [(C, K)], [N], [B], [0], cls, base_cost, {"seed": seed, "c_max": cm})


# ----------------------------------------------------------------------------- NEXT-4 inputs
def supermodular_gain_table(K: int, C: int = NUM_CLASSES) -> np.ndarray:
    """NEXT-4 profile: g[c][k] = A_c * H_k (units of 0.001 mAP point), A_c = round(1400 *
    0.604**(9-c)) (Appendix-B amplitude), H_0 = 0, H_k = round(10 * (0.561 +
    0.439 (k-1)/(K-2))). Both factors are non-decreasing integers, so the table has increasing
    differences in the class exactly (reading R19)."""
    A = [int(math.floor(1400.0 * 0.604 ** (9 - c) + 0.5)) for c in range(C)]
    H = [0] + [int(math.floor(10.0 * (1.0 if K == 2 else 0.561 + 0.439 * (k - 1) / (K - 2)) + 0.5))
               for k in range(1, K)]
    return np.array([[A[c] * H[k] for k in range(K)] for c in range(C)], dtype=np.int32).reshape(-1)


def batch_latency_table(K: int, c_max: int, cap: int) -> np.ndarray:
    """I_k(n) for n = 0..cap: 0 for an empty batch, else ceil(c_k (2 + 3n) / 5) -- a fixed 40 %
    launch share plus 60 % per frame (a batch of n frames costs less than n singles, the reason
    the paper batches same-level frames), c_k = ceil(c_max k / (K-1))."""
    ck = regular_costs(K, c_max)
    t = np.zeros((K, cap + 1), dtype=np.int64)
    for k in range(K):
        for n in range(1, cap + 1):
            t[k, n] = -((-int(ck[k]) * (2 + 3 * n)) // 5)
    return t.reshape(-1).astype(np.int32)


BATCHED_CONFIGS = {
    1: dict(W=1, N=30, K=4, B=120),
    2: dict(W=1024, N=30, K=5, B=1000),
}


def make_batched_config(k: int, num_windows: Optional[int] = None, window_offset: int = 0) -> Workload:
    """NEXT-4 workload b<k>: the c<k> window shapes and class mix, batched latency tables."""
    p = BATCHED_CONFIGS[k]
    W = p["W"] if num_windows is None else num_windows
    N, K, B = p["N"], p["K"], p["B"]
    seed = BASE_SEED + 100 + k
    wid = np.arange(window_offset, window_offset + W, dtype=np.int64)
    nf = np.full(W, N, dtype=np.int32)
    cls = _class_ids(seed, nf, np.full(W, 0.35), window_ids=wid)
    c_max = -((-3 * B) // N)
    g = supermodular_gain_table(K)
    wl = _wl(f"b{k}", [g], [np.tile(regular_costs(K, c_max), NUM_CLASSES).astype(np.int32)], [(NUM_CLASSES, K)],
             nf, np.full(W, B), np.zeros(W), cls, 84, {"config": f"b{k}", "N": N, "K": K, "B": B, "c_max": c_max})
    wl.profiles_batch = [batch_latency_table(K, c_max, N)]
    wl.batch_cap = N
    return wl


def make_batched_random(seed: int, W: int, max_frames: int = 8, K: int = 3, C: int = 4, max_budget: int = 40,
                        linear: bool = False, general: bool = False) -> Workload:
    """Parity set for NEXT-4: random supermodular gains (negative entries allowed), random
    non-decreasing batch tables (or linear ones, I_k(n) = n c_k, when `linear`), random budgets
    including infeasible windows (I_0(n) > 0 in some profiles). general: gains U{-4..12} with no
    structure at all (most profiles then violate R19; small ranges give many ties)."""
    wid = np.arange(W, dtype=np.int64)
    nf = rand_int(seed, S_TN, wid, 0, max_frames).astype(np.int32)
    bud = rand_int(seed, S_TBUD, wid, 0, max_budget).astype(np.int32)
    cap = max_frames
    gains, costs, batches, shapes = [], [], [], []
    P = 8
    for q in range(P):
        # A_c and H_k non-decreasing integers (possibly negative offsets): g = A_c H_k + r_k
        A = np.cumsum(rand_int(seed, S_TGAIN * 97 + q, np.arange(C), 0, 3)) - 2
        H = np.cumsum(rand_int(seed, S_TGAIN * 89 + q, np.arange(K), 0, 3))
        r = rand_int(seed, S_TGAIN * 83 + q, np.arange(K), -3, 3)
        g = (A[:, None] * H[None, :] + r[None, :]).astype(np.int32).reshape(-1)
        if general:
            g = rand_int(seed, S_TGAIN * 79 + q, np.arange(C * K), -4, 12).astype(np.int32)
        ck = rand_int(seed, S_TCOST * 97 + q, np.arange(K), 0, 6)
        fixed = rand_int(seed, S_TBASE * 97 + q, np.arange(K), 0, 4)
        t = np.zeros((K, cap + 1), dtype=np.int64)
        for k in range(K):
            for n in range(1, cap + 1):
                t[k, n] = n * ck[k] if linear else fixed[k] + n * ck[k] - (n // 3)
            t[k] = np.maximum.accumulate(t[k])
        if not linear and q % 3 == 0:
            t[0, 1:] += 1                                         # I_0(n) > 0: infeasible windows
        gains.append(g)
        costs.append(np.tile(ck, C).astype(np.int32))
        batches.append(t.reshape(-1).astype(np.int32))
        shapes.append((C, K))
    prof = rand_int(seed, S_PROF, wid, 0, P - 1).astype(np.int32)
    F = int(nf.sum())
    cls = rand_int(seed, S_CLASS, np.arange(F, dtype=np.int64), 0, C - 1).astype(np.uint8)
    wl = _wl(f"batched_random_{seed}", gains, costs, shapes, nf, bud, prof, cls, 0)
    wl.profiles_batch = batches
    wl.batch_cap = cap
    return wl


# ----------------------------------------------------------------------------- NEXT-5 parity sets
S_NN_GAIN, S_NN_COST, S_NN_ZERO, S_NN_N, S_NN_B, S_NN_PROF, S_NN_NOZ = range(50, 57)


def make_nonneg_set(seed: int, W: int, K: int, max_frames: int, min_budget: int, max_budget: int,
                    max_gain: int, max_cost: int, num_profiles: int = 8, C: int = NUM_CLASSES,
                    no_zero_frac: float = 0.0, base_cost: int = 5) -> Workload:
    """Windows of ONE K with gains U{0..max_gain} and costs U{0..max_cost}, where in every class
    row one exit (drawn per row, not always exit 0) costs 0 -- the shape of the paper's tables
    (gains >= 0, the no-enhancement exit free) that the u16 rows of NEXT-5 serve. A fraction
    `no_zero_frac` of the profiles keeps no cost-0 exit (those windows stay on int32 rows).
    Budgets U{min_budget..max_budget}, N U{0..max_frames}. Inputs only."""
    gains, costs, shapes = [], [], []
    for p in range(num_profiles):
        n = C * K
        g = rand_int(seed, S_NN_GAIN, p * 4096 + np.arange(n), 0, max_gain).astype(np.int32)
        c = rand_int(seed, S_NN_COST, p * 4096 + np.arange(n), 0, max_cost).astype(np.int32)
        if rand_uniform(seed, S_NN_NOZ, p) >= no_zero_frac:
            z = rand_int(seed, S_NN_ZERO, p * 64 + np.arange(C), 0, K - 1)
            c.reshape(C, K)[np.arange(C), z] = 0
        else:
            c = np.maximum(c, 1).astype(np.int32)
        gains.append(g)
        costs.append(c)
        shapes.append((C, K))
    wid = np.arange(W)
    N = rand_int(seed, S_NN_N, wid, 0, max_frames).astype(np.int32)
    B = rand_int(seed, S_NN_B, wid, min_budget, max_budget).astype(np.int32)
    prof = rand_int(seed, S_NN_PROF, wid, 0, num_profiles - 1).astype(np.int32)
    u = rand_uniform(seed, S_CLASS, np.arange(int(N.sum())))
    cls = np.minimum((u * C).astype(np.int64), C - 1)
    return _wl(f"nonneg{seed}_K{K}", gains, costs, shapes, N, B, prof, cls, base_cost, {"seed": seed})


def make_u16_boundary(y: int, base_cost: int = 5) -> Workload:
    """One window at the edge of the u16 row rule (NEXT-5): 21 frames, K = 4, costs (0, 1, 2, 3),
    20 frames with gains (0, 1, 2, 3000) and one with (0, 1, 2, y), budget 63 (every frame can
    take exit 3), and the same frames under budgets 40, 17 and 0. sum_i max_k g + max g + 1 =
    63001 + y: y = 2534 is exactly 65535 (u16 rows), y = 2535 one above (int32 rows). Inputs only."""
    g = np.array([0, 1, 2, 3000, 0, 1, 2, y], dtype=np.int32)
    c = np.array([0, 1, 2, 3, 0, 1, 2, 3], dtype=np.int32)
    cls = np.array(([0] * 10 + [1] + [0] * 10) * 4, dtype=np.int64)
    return _wl(f"u16_boundary_{y}", [g], [c], [(2, 4)], [21] * 4, [63, 40, 17, 0], [0] * 4, cls, base_cost,
               {"y": y})


# ----------------------------------------------------------------------------- a1 edge inputs
S_EDGE_MODE, S_EDGE_VAL = 40, 41


def with_budget_edges(wl: Workload, seed: int) -> Workload:
    """Copy of `wl` whose capacities exercise every branch of a1 (reading R3):
    the layout bound stays wl.budget, while the capacity handed to the path is drawn per window:
      25 %  capacity in [N u0 - 100, N u0]   -> a1 clamps (budget 0; exactly 0 when = N u0)
      10 %  capacity in [-1000, N u0]        -> deep clamp, some capacities negative
      35 %  capacity = N u0 + U{0..B_bound}  -> device budget below (or at) the layout bound
      30 %  unchanged (capacity = N u0 + B_bound, the exact fit)
    Inputs only: no budget is computed here (the code under test derives it)."""
    W = wl.num_windows
    wid = np.arange(W, dtype=np.int64)
    u = rand_uniform(seed, S_EDGE_MODE, wid)
    nu0 = wl.num_frames.astype(np.int64) * int(wl.base_cost)
    bb = wl.budget.astype(np.int64)
    r = rand_uniform(seed, S_EDGE_VAL, wid)
    cap = wl.capacity.astype(np.int64).copy()
    m1 = u < 0.25
    cap[m1] = nu0[m1] - np.floor(r[m1] * 101).astype(np.int64)
    m2 = (u >= 0.25) & (u < 0.35)
    cap[m2] = -1000 + np.floor(r[m2] * (nu0[m2] + 1001)).astype(np.int64)
    m3 = (u >= 0.35) & (u < 0.70)
    cap[m3] = nu0[m3] + np.floor(r[m3] * (bb[m3] + 1)).astype(np.int64)
    out = Workload(f"{wl.name}+edges{seed}", wl.profiles_gain, wl.profiles_cost, wl.profiles_shape,
                   wl.num_frames.copy(), wl.budget.copy(), cap.astype(np.int32), wl.base_cost, wl.profile.copy(),
                   wl.class_id.copy(), dict(wl.meta))
    return out

"""Window sharding across GPUs: windows are independent, so a
rank owns a contiguous window range and the only collective is the stats allreduce."""
from __future__ import annotations

import numpy as np


def work_per_window(num_frames, budget, num_exits) -> np.ndarray:
    """DP work of each window: N_w (B_w + 1) K_w max-plus evaluations."""
    return (np.asarray(num_frames, np.int64) * (np.asarray(budget, np.int64) + 1)
            * np.asarray(num_exits, np.int64))


def shard_ranges(work, world: int):
    """Contiguous [lo, hi) window ranges, one per rank, balanced by cumulative work.

    Rank r takes the windows whose work prefix midpoint falls in [r, r+1) * total / world, so
    every window belongs to exactly one rank and the ranges are ordered by rank."""
    work = np.asarray(work, dtype=np.float64)
    W = len(work)
    if world <= 1 or W == 0:
        return [(0, W)] + [(W, W)] * max(world - 1, 0)
    if work.sum() <= 0:
        work = np.ones(W, dtype=np.float64)             # no work anywhere: balance counts
    cum = np.cumsum(work)
    total = cum[-1]
    mid = cum - work / 2.0
    owner = np.minimum((mid * world / total).astype(np.int64), world - 1)
    bounds = np.searchsorted(owner, np.arange(world + 1), side="left")
    return [(int(bounds[r]), int(bounds[r + 1])) for r in range(world)]

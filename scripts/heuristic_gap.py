#!/usr/bin/env python
"""NEXT-1 measurement: the paper's prune-and-search heuristic (turbo_heuristic_plan) against the
exact DP (turbo_mckp_solve, the paper's "upper") on the same windows, on one B200.
Prints one JSON line per workload: mean / max relative gain gap, windows where the heuristic
is suboptimal, and both kernels' device times (CUDA events, graph-free, L2 not flushed)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(name, wl, reps=5):
    import numpy as np
    import torch
    from paper_2207_00172_b200 import turbo
    b = turbo.batch_from_workload(wl)
    turbo.run_path(b, fused=True)
    W = wl.num_windows
    dev = b.best_gain.device
    hg = torch.zeros(W, dtype=torch.int32, device=dev)
    hc = torch.zeros(W, dtype=torch.int32, device=dev)
    hf = torch.zeros(W, dtype=torch.uint8, device=dev)
    hs = torch.zeros(W, dtype=torch.int32, device=dev)
    hx = torch.zeros(max(wl.total_frames, 1), dtype=torch.uint8, device=dev)

    def t_of(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    t_h = t_of(lambda: turbo.heuristic_plan(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, hg, hc, hf, hx, hs))
    t_e = t_of(lambda: turbo.mckp_solve(b.shape, b.windows_dev, b.opt_gain, b.opt_cost, b.solve_ws, b.best_gain,
                                        b.best_cost, b.feasible, b.exit_out, b.status))
    eg = b.best_gain[:W].cpu().numpy().astype(np.int64)
    ef = b.feasible[:W].cpu().numpy()
    g = hg.cpu().numpy().astype(np.int64)
    f = hf.cpu().numpy()
    ok = (ef == 1) & (f == 1) & (eg > 0)
    gap = (eg[ok] - g[ok]) / eg[ok]
    return {"workload": name, "windows": W, "mean_gap": float(gap.mean()) if ok.any() else 0.0,
            "max_gap": float(gap.max()) if ok.any() else 0.0, "suboptimal_windows": int((gap > 0).sum()),
            "heuristic_infeasible_where_exact_feasible": int(((ef == 1) & (f == 0)).sum()),
            "mean_downgrade_steps": float(hs.cpu().numpy().mean()),
            "t_heuristic_ms": t_h, "t_exact_ms": t_e, "exact_dominates": bool((eg[ok] >= g[ok]).all())}


def main():
    import synth
    cases = [("c2", synth.make_config(2)), ("c3-shard", synth.make_config(3, num_windows=8192)),
             ("c5-shard", synth.make_config(5, num_windows=2048)),
             ("tie-heavy", synth.make_tie_heavy(seed=44, W=4096, max_frames=60, max_exits=8, max_budget=150))]
    for name, wl in cases:
        print(json.dumps(run(name, wl)), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Small cases through every kernel path, for compute-sanitizer (one tool per run):
the per-class CTA kernels (fused / plan / smem / HBM variants), the runtime-K kernel, the
lockstep kernel, the long-row cluster kernel, the long-window grid kernel on both its paths (halo segments and L2 rows) with
its walk kernel, the u16-row kernels (NEXT-5), turbo_schedule_theta, the batches / latency kernel and
both NEXT-4 kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import synth
    from paper_2207_00172_b200 import turbo
    turbo.load()
    long2 = synth.concat_workloads([synth.make_long_window(4, N=12, K=5, B=30000),
                                    synth.make_long_window(5, N=9, K=4, B=26000, c_max=5000, random_rows=True)])
    cases = [synth.make_config(1), synth.make_config(2, num_windows=16),
             synth.make_tie_heavy(seed=9, W=64, max_frames=12, max_exits=9, max_budget=700),
             synth.make_config(5, num_windows=24), long2]
    for wl in cases:
        for fused, variant in ((True, 0), (True, 1), (True, 2), (False, 0), (True, 4), ("all", 0), ("all", 32),
                               (True, 512), ("all", 512)):
            turbo.debug_set_variant(variant)
            b = turbo.batch_from_workload(wl, with_plan_workspace=True)
            turbo.run_path(b, fused=fused)
            torch.cuda.synchronize()
            turbo.debug_set_variant(0)
    # lockstep kernel (variant 8) on a c2-shaped batch of >= 2 windows per SM
    turbo.debug_set_variant(8)
    b = turbo.batch_from_workload(synth.make_config(2, num_windows=400))
    turbo.run_path(b, fused="all")
    torch.cuda.synchronize()
    turbo.debug_set_variant(0)
    # NEXT-5 u16 rows (variant 128): in-place and multi-warp rows, shifts beyond the pad, fused and solve
    wl = synth.make_nonneg_set(seed=5, W=60, K=5, max_frames=30, min_budget=0, max_budget=4000, max_gain=1400,
                               max_cost=901, no_zero_frac=0.3)
    for fused in ("all", True):
        turbo.debug_set_variant(128)
        b = turbo.batch_from_workload(wl, with_plan_workspace=False)
        turbo.run_path(b, fused=fused)
        torch.cuda.synchronize()
        turbo.debug_set_variant(0)
    # NEXT-3 fused, NEXT-2 latency
    wl = synth.make_config(5, num_windows=24)
    b = turbo.batch_from_workload(wl, with_plan_workspace=False)
    th = torch.rand(wl.total_frames, device="cuda")
    cls = torch.zeros(wl.total_frames, dtype=torch.uint8, device="cuda")
    turbo.schedule_theta(b.shape, b.profiles_dev, b.windows_dev, th, 0.1, cls, b.capacity, b.base_cost, b.solve_ws,
                         b.best_gain, b.best_cost, b.feasible, b.exit_out, b.stats, b.status)
    W, F = wl.num_windows, wl.total_frames
    cnt = torch.zeros(16 * W, dtype=torch.int32, device="cuda")
    order = torch.zeros(F, dtype=torch.int32, device="cuda")
    cap = int(wl.num_frames.max())
    tabs = [np.zeros(K * (cap + 1), np.int32) for (C, K) in wl.profiles_shape]
    bt = turbo.batch_cost_table(tabs, wl.profiles_shape, cap)
    lat = torch.zeros(W, dtype=torch.int64, device="cuda")
    turbo.batches(b.shape, b.windows_dev, b.exit_out, cnt, order, bt, cap, lat, b.status)
    torch.cuda.synchronize()
    # NEXT-4: enumeration + the general program (variant 64 forces it)
    for variant in (0, 64):
        wl = synth.make_batched_random(3, 40, max_frames=8, K=4, C=4, max_budget=50, general=True)
        b = turbo.make_batch(wl.profiles_gain, wl.profiles_cost, wl.profiles_shape, wl.num_frames, wl.budget,
                             wl.profile, class_id=wl.class_id, with_plan_workspace=False)
        bt = turbo.batch_cost_table(wl.profiles_batch, wl.profiles_shape, wl.batch_cap)
        n = turbo.batched_workspace(b.shape)
        ws = torch.empty(max(n, 16), dtype=torch.uint8, device="cuda")
        turbo.debug_set_variant(variant)
        turbo.batched_plan(b.shape, b.windows_dev, b.profiles_dev, bt, wl.batch_cap, b.class_id, b.best_gain,
                           b.best_cost, b.feasible, b.exit_out, b.status, workspace=ws)
        torch.cuda.synchronize()
        turbo.debug_set_variant(0)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()

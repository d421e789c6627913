#!/usr/bin/env python
"""Per-call device times of the hot path (CUDA events around each C-ABI call, L2 warm):
lookup, solve (a3-a5 fused), plan (a3+a4), backtrack (a5), stats (a6), schedule (a1-a6)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--windows", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    import synth
    from paper_2207_00172_b200 import turbo
    import bench
    spec = bench.WORKLOADS[args.workload]
    n = args.windows or spec["per_gpu"]
    wl = synth.make_config(spec["config"], num_windows=n)
    b = turbo.batch_from_workload(wl, with_plan_workspace=True)
    s = b.shape
    calls = {
        "lookup": lambda: turbo.profile_lookup(s, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost,
                                               b.opt_gain, b.opt_cost, b.status),
        "solve": lambda: turbo.mckp_solve(s, b.windows_dev, b.opt_gain, b.opt_cost, b.solve_ws, b.best_gain,
                                          b.best_cost, b.feasible, b.exit_out, b.status),
        "plan": lambda: turbo.mckp_plan(s, b.windows_dev, b.opt_gain, b.opt_cost, b.workspace, b.best_gain,
                                        b.best_cost, b.feasible, b.status),
        "backtrack": lambda: turbo.backtrack(s, b.windows_dev, b.opt_cost, b.workspace, b.best_cost, b.feasible,
                                             b.exit_out),
        "stats": lambda: turbo.stats(s, b.windows_dev, b.class_id, b.exit_out, b.best_gain, b.best_cost,
                                     b.feasible, b.stats),
    }
    if int(s.num_big) == 0:
        calls["schedule"] = lambda: turbo.schedule(s, b.profiles_dev, b.windows_dev, b.class_id, b.capacity,
                                                   b.base_cost, b.solve_ws, b.best_gain, b.best_cost, b.feasible,
                                                   b.exit_out, b.stats, b.status)
    for name, fn in calls.items():
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        print(f"{args.workload} {name:10s} median {ts[len(ts) // 2]:9.4f} ms  min {ts[0]:9.4f} ms", flush=True)
    st = b.status.cpu().numpy()
    print("status", st.tolist())


if __name__ == "__main__":
    main()

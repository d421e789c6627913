#!/usr/bin/env python
"""Run the hot path on one workload a few times (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--windows", type=int, default=0, help="0 = bench.py's per-GPU share")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--path", choices=["schedule", "solve", "plan"], default="schedule")
    ap.add_argument("--variant", type=int, default=0)
    args = ap.parse_args()
    import torch
    import synth
    from paper_2207_00172_b200 import turbo
    import bench
    spec = bench.WORKLOADS[args.workload]
    n = args.windows or spec["per_gpu"]
    wl = synth.make_config(spec["config"], num_windows=n)
    turbo.debug_set_variant(args.variant)
    b = turbo.batch_from_workload(wl, with_plan_workspace=args.path == "plan" or (args.variant & 3) == 2)
    fused = {"schedule": "all", "solve": True, "plan": False}[args.path]
    for _ in range(args.reps):
        turbo.run_path(b, fused=fused)
    torch.cuda.synchronize()
    st = b.status.cpu().numpy()
    assert st[0] == -1 and st[1] == -1, st
    print("ok", args.workload, n, "windows")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Small cases through every kernel path, for compute-sanitizer (one tool per run)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synth
    from paper_2207_00172_b200 import turbo
    cases = [synth.make_config(1), synth.make_config(2, num_windows=16),
             synth.make_tie_heavy(seed=9, W=64, max_frames=12, max_exits=9, max_budget=700),
             synth.make_config(5, num_windows=24), synth.make_long_window(4, N=20, K=5, B=30000)]
    for wl in cases:
        long_rows = bool((wl.budget.astype(int) + 1 > 24576).any())
        for fused, variant in ((True, 0), (True, 1), (True, 2), (False, 0), (True, 4), ("all", 0)):
            if long_rows and fused == "all":
                continue                      # turbo_schedule does not serve long windows
            turbo.debug_set_variant(variant)
            b = turbo.batch_from_workload(wl, with_plan_workspace=True)
            turbo.run_path(b, fused=fused)
            torch.cuda.synchronize()
            turbo.debug_set_variant(0)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()

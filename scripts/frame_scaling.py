#!/usr/bin/env python
"""Kernel time of turbo_schedule on c2-shaped batches (1024 windows, K=5, B=1000) as a function of
the frame count N: the intercept is the per-window prologue/epilogue, the slope the per-frame cost."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synth
    from synth.workloads import _uniform_config
    from paper_2207_00172_b200 import turbo
    for N in (1, 2, 4, 8, 16, 30, 60):
        wl = _uniform_config(2, 1024, N, 5, 1000)
        b = turbo.batch_from_workload(wl)
        fn = lambda: turbo.schedule(b.shape, b.profiles_dev, b.windows_dev, b.class_id, b.capacity, b.base_cost,
                                    b.solve_ws, b.best_gain, b.best_cost, b.feasible, b.exit_out, b.stats, b.status)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"N={N:3d} schedule kernel {e0.elapsed_time(e1) / 20 * 1e3:8.2f} us")


if __name__ == "__main__":
    main()

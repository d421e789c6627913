#!/usr/bin/env python
"""Experiment: the launch order of the row-size class launches (turbo_shape_t.cls_order) on a
multi-class batch (default c5): time turbo_schedule per order with CUDA events (graph replay)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import json
    import torch
    import synth
    from paper_2207_00172_b200 import turbo
    turbo.load()
    wl = synth.make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
    b = turbo.batch_from_workload(wl, with_plan_workspace=False)
    res = {}
    orders = [0x3210, 0x0123, 0x2103, 0x1023, 0x0213]
    for rep in range(2):
        for o in orders:
            b.shape.cls_order = o
            g = torch.cuda.CUDAGraph()
            turbo.run_path(b, fused="all")
            torch.cuda.synchronize()
            with torch.cuda.graph(g):
                turbo.run_path(b, fused="all")
            for _ in range(2):
                g.replay()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            for _ in range(5):
                g.replay()
            ev[1].record()
            torch.cuda.synchronize()
            res.setdefault(hex(o), []).append(ev[0].elapsed_time(ev[1]) / 5)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Long rows beyond one CTA (TURBO_BIG_CELLS < cells <= TURBO_CLUSTER_CELLS): the cluster kernel
(default) against the grid kernel (variant 512) on the same batch -- device time of one
turbo_schedule call (CUDA graph replay, CUDA events), and bit-equality of the two outputs.
usage: scripts/cluster_vs_grid.py [W] [N] [K] [B]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import synth
    from paper_2207_00172_b200 import turbo
    W, N, K, B = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (64, 300, 6, 60000)))
    turbo.load()
    wl = synth.concat_workloads([synth.make_long_window(500 + s, N=N, K=K, B=B) for s in range(W)])
    out = {"windows": W, "frames": N, "exits": K, "budget": B, "cells": int(wl.total_cells)}
    res = {}
    for name, variant in (("cluster", 0), ("grid", 512)):
        turbo.debug_set_variant(variant)
        b = turbo.batch_from_workload(wl, with_plan_workspace=False)
        turbo.run_path(b, fused="all")
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            turbo.run_path(b, fused="all")
        g.replay()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        reps = 3
        ev[0].record()
        for _ in range(reps):
            g.replay()
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        res[name] = turbo.results(b)
        out[name] = {"ms": ms, "cell_updates_per_s": wl.total_cells / (ms / 1e3)}
        turbo.debug_set_variant(0)
    same = all(np.array_equal(res["cluster"][k], res["grid"][k]) for k in ("exits", "best_gain", "best_cost", "feasible"))
    out["identical_outputs"] = bool(same)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

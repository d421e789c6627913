#!/usr/bin/env python
"""Per-CTA phase timeline of the fused schedule kernel (turbo_debug_trace, %globaltimer ns):
CTA start, prologue, DP, optimum, plan reconstruction, end -- on bench.py's workload shape."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--path", choices=["schedule", "solve"], default="schedule")
    args = ap.parse_args()
    import numpy as np
    import torch
    import synth
    import bench
    from paper_2207_00172_b200 import turbo
    spec = bench.WORKLOADS[args.workload]
    wl = synth.make_config(spec["config"], num_windows=spec["per_gpu"])
    b = turbo.batch_from_workload(wl)
    fused = "all" if args.path == "schedule" else True
    for _ in range(3):
        turbo.run_path(b, fused=fused)
    torch.cuda.synchronize()
    buf = torch.zeros(8 * 65536, dtype=torch.int64, device="cuda")
    turbo.debug_trace(buf)
    turbo.run_path(b, fused=fused)
    torch.cuda.synchronize()
    turbo.debug_trace(None)
    tr = buf.view(-1, 8).cpu().numpy()
    tr = tr[tr[:, 0] > 0]
    t0 = tr[:, 0].min()
    names = ["start", "prologue", "dp", "optimum", "backtrack", "end"]
    print(f"{args.workload}: {len(tr)} CTAs traced; times in us relative to the first CTA start")
    rel = (tr[:, :6] - t0) / 1e3
    for p, nm in enumerate(names):
        v = rel[:, p]
        print(f"  {nm:10s} at   min {v.min():8.2f}  median {np.median(v):8.2f}  max {v.max():8.2f}")
    for p in range(1, 6):
        d = (tr[:, p] - tr[:, p - 1]) / 1e3
        print(f"  {names[p - 1]}->{names[p]:10s} median {np.median(d):7.2f} us  p90 {np.percentile(d, 90):7.2f}"
              f"  max {d.max():7.2f}")
    tot = (tr[:, 5] - tr[:, 0]) / 1e3
    print(f"  CTA lifetime median {np.median(tot):.2f} us, kernel span {rel[:, 5].max():.2f} us")


if __name__ == "__main__":
    main()

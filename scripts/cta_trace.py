#!/usr/bin/env python
"""Per-window phase timeline of the CTA DP kernels (turbo_debug_trace, %globaltimer ns; needs a
library built with the trace marks: TURBO_TRACE=1 python -c "from paper_2207_00172_b200 import build;
build.build(force=True)"):
window start, prologue, DP, optimum, in-kernel plan reconstruction, end -- per row-size class,
on bench.py's workload shape."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BOUNDS = (256, 1024, 4608, 24576)


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
    W = int(b.shape.num_windows)
    buf = torch.zeros(8 * W, dtype=torch.int64, device="cuda")
    turbo.debug_trace(buf)
    turbo.run_path(b, fused=fused)
    torch.cuda.synchronize()
    turbo.debug_trace(None)
    tr = buf.view(W, 8).cpu().numpy().astype(np.float64)
    wins = b.windows_host
    cells = wins["budget_bound"].astype(np.int64) + 1
    cls = np.searchsorted(np.array(BOUNDS), cells, side="left")
    work = wins["num_frames"].astype(np.int64) * cells * (wins["num_exits"].astype(np.int64) + 1)
    ok = tr[:, 0] > 0
    t0 = tr[ok, 0].min()
    rel = (tr - t0) / 1e3
    print(f"{args.workload} ({args.path}): {ok.sum()} of {W} windows traced; us from the first window start")
    print(f"  kernel span (last window end) {rel[ok, 5].max():.1f} us")
    for c in range(5):
        m = ok & (cls == c)
        if not m.any():
            continue
        dp = (tr[m, 2] - tr[m, 1]) / 1e3
        pro = (tr[m, 1] - tr[m, 0]) / 1e3
        life = (tr[m, 5] - tr[m, 0]) / 1e3
        print(f"  class {c}: {m.sum():5d} windows  start [{rel[m, 0].min():8.1f} .. {rel[m, 0].max():8.1f}]"
              f"  end max {rel[m, 5].max():8.1f}  prologue med {np.median(pro):6.2f}  dp med {np.median(dp):8.1f}"
              f" max {dp.max():8.1f}  life max {life.max():8.1f}")
        heavy = np.argsort(-work[m])[:3]
        idx = np.nonzero(m)[0][heavy]
        for w in idx:
            print(f"      heavy window {w}: N={wins['num_frames'][w]} B={wins['budget_bound'][w]} "
                  f"K={wins['num_exits'][w]} start {rel[w, 0]:.1f} end {rel[w, 5]:.1f} life {rel[w, 5] - rel[w, 0]:.1f}")
    if args.workload == "c2":
        names = ["start", "prologue", "dp", "optimum", "backtrack", "end"]
        for p in range(1, 6):
            d = (tr[ok, p] - tr[ok, p - 1]) / 1e3
            print(f"  {names[p - 1]}->{names[p]:10s} median {np.median(d):7.2f} us  p90 {np.percentile(d, 90):7.2f}"
                  f"  max {d.max():7.2f}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-CTA cycle counters of the long-window grid kernel (TURBO_GRID_DEBUG=2) on config c4."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["TURBO_GRID_DEBUG"] = os.environ.get("TURBO_GRID_DEBUG", "2")


def main():
    import numpy as np
    import torch
    import synth
    from paper_2207_00172_b200 import turbo
    wl = synth.make_config(4)
    b = turbo.batch_from_workload(wl)
    turbo.run_path(b, fused=True)
    torch.cuda.synchronize()
    ws = b.solve_ws.cpu().numpy()
    off = int(b.shape.grid_scratch_offset)
    tr = ws[off + 4 * (2 * 256 + 64): off + 4 * (2 * 256 + 64) + 8 * 8 * 256].view(np.int64).reshape(256, 8)[:148]
    names = ["retries", "consume", "ship", "step", "mbar_wait", "to_consume", "-", "steps"]
    steps = np.maximum(tr[:, 7], 1)
    for k in (0, 1, 2, 3, 4, 5):
        per = tr[:, k] / steps
        print(f"{names[k]:8s} per step: mean {per.mean():10.1f} min {per.min():10.1f} max {per.max():10.1f}"
              + ("" if k == 0 else "  (cycles)"))
    for j in (0, 1, 2, 73, 145, 146, 147):
        print(j, (tr[j, :6] / steps[j]).round(1).tolist(), int(tr[j, 7]))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Copy one measurement pass (scripts/round_measure.sh, gpurun_out/round/) into profiles/ with a
round prefix: bench lines, the launch list, ncu summaries (+ details CSV) and the per-workload DRAM
traffic files bench.py reports as roofline.traffic.

usage: scripts/collect_round.py r02 [DEST_DIR]   (default profiles/; on a GPU box use a directory
under gpurun_out/ -- only gpurun_out/ travels back)"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "round")
DST = os.path.join(ROOT, "profiles")
TRAFFIC = {"full_schedule_c2": "c2", "full_schedule_c3": "c3", "full_grid_c4": "c4",
           "full_schedule_c5_cls3": "c5", "full_batched_b2": "b2", "full_cluster_lw": "lw"}


def main():
    global DST
    tag = sys.argv[1]
    if len(sys.argv) > 2:
        DST = sys.argv[2]
        os.makedirs(DST, exist_ok=True)
    for f in sorted(os.listdir(SRC)):
        p = os.path.join(SRC, f)
        if f.startswith("bench_") and f.endswith(".json"):
            lines = [ln for ln in open(p).read().splitlines() if ln.startswith("{")]
            if lines:
                with open(os.path.join(DST, f"{tag}_{f}"), "w") as o:
                    o.write(lines[-1] + "\n")
        elif f == "launches_c2.csv":
            shutil.copy(p, os.path.join(DST, f"{tag}_launches_c2.csv"))
        elif f.endswith(".ncu-rep"):
            name = f[:-8]
            args = [sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), p, f"{tag}_ncu_{name}",
                    TRAFFIC.get(name, name), "", DST]
            r = subprocess.run(args, capture_output=True, text=True)
            if r.returncode != 0:
                print("summary failed", f, r.stderr[-500:])
            if name not in TRAFFIC:           # only the dominant kernels feed roofline.traffic
                tf = os.path.join(DST, f"traffic_{name}.json")
                if os.path.exists(tf):
                    os.remove(tf)
    print("collected into profiles/ with prefix", tag)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Summarise an `ncu --set full` report of one kernel launch into profiles/: key metrics (JSON),
the details page (CSV), and the DRAM traffic per launch that bench.py reports as
roofline.traffic (profiles/traffic_<workload>.json).

usage: scripts/ncu_summary.py REPORT.ncu-rep NAME WORKLOAD [KERNEL_LABEL] [DEST_DIR]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "sm__cycles_elapsed.avg.per_second", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "launch__occupancy_limit_shared_mem", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
] + [f"smsp__average_warps_issue_stalled_{r}_per_issue_active.ratio" for r in (
    "barrier", "branch_resolving", "dispatch_stall", "drain", "lg_throttle", "long_scoreboard",
    "math_pipe_throttle", "membar", "mio_throttle", "misc", "no_instruction", "not_selected", "selected",
    "short_scoreboard", "sleeping", "tex_throttle", "wait")]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"Kernel Name": vals[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = f"{vals[i]} {units[i]}".strip()
    return d


def to_bytes(s):
    v, _, u = s.partition(" ")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u.strip(), 1)
    return float(v.replace(",", "")) * scale


def main():
    rep, name, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    label = sys.argv[4] if len(sys.argv) > 4 else ""
    d = raw(rep)
    prof = sys.argv[5] if len(sys.argv) > 5 else os.path.join(ROOT, "profiles")
    with open(os.path.join(prof, f"{name}_summary.json"), "w") as f:
        json.dump(d, f, indent=1)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    with open(os.path.join(prof, f"{name}_details.csv"), "w") as f:
        f.write(det)
    traffic = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
    with open(os.path.join(prof, f"traffic_{workload}.json"), "w") as f:
        json.dump({"workload": workload, "kernel": label or d["Kernel Name"], "dram_bytes_per_launch": traffic,
                   "source": f"profiles/{name}_summary.json (ncu --set full, one launch)"}, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()

#!/bin/bash
# ncu launch list (device time per kernel) of one bench step: $1 workload, $2 variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
W=$1; V=${2:-0}
python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --variant $V > gpurun_out/launch_${W}_v$V.plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic,sm__warps_active.avg.per_cycle_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio \
    --clock-control none -k regex:'dp_|walk_|lookup_|stats_|backtrack_' -c 12 --csv --log-file gpurun_out/launch_${W}_v$V.csv \
    python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline --variant $V > gpurun_out/launch_${W}_v$V.ncu.log 2>&1

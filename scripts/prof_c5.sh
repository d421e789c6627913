#!/bin/bash
# c5: per-launch device times of one turbo_schedule step (ncu launch list) + ncu --set full of the
# longest DP class kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__shared_mem_per_block_dynamic,launch__registers_per_thread,sm__warps_active.avg.per_cycle_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:'dp_|walk_|lookup_|stats_' -c 40 --csv --log-file gpurun_out/c5_launches.csv \
    python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_ncu1.log 2>&1
#ncu --set full --clock-control none --import-source on -k regex:'dp_cta_kernel' -s 3 -c 1 \
#    -o gpurun_out/prof_c5_cls3 -f python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_ncu2.log 2>&1

#!/bin/bash
# ncu --set full with the SASS source page of one kernel of one bench workload (summarised on the
# box: raw metrics CSV + per-instruction SASS CSV; the report itself is dropped).
# usage: scripts/prof_src.sh NAME WORKLOAD KERNEL_REGEX SKIP [extra bench args]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
N=$1; W=$2; K=$3; S=$4; shift 4
mkdir -p gpurun_out/src
python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/src/plain_$N.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -o gpurun_out/src/$N -f \
    python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/src/ncu_$N.log 2>&1
ncu -i gpurun_out/src/$N.ncu-rep --page raw --csv > gpurun_out/src/raw_$N.csv 2>&1
ncu -i gpurun_out/src/$N.ncu-rep --page source --csv --print-source sass > gpurun_out/src/sass_$N.csv 2>&1
ncu -i gpurun_out/src/$N.ncu-rep --page source --csv --print-source cuda > gpurun_out/src/cuda_$N.csv 2>&1
rm -f gpurun_out/src/$N.ncu-rep

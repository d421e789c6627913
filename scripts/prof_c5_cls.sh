#!/bin/bash
# ncu --set full of one c5 class kernel: $1 = dp_cta_kernel launches to skip (class = $1 mod 4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_plain.log 2>&1 && \
for s in "$@"; do
ncu --set full --clock-control none --import-source on -k regex:'dp_cta_kernel' -s $s -c 1 \
    -o gpurun_out/prof_c5_s$s -f python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c5_ncu_s$s.log 2>&1
done

#!/bin/bash
# ncu --set full of the c2 DP kernel: lockstep (variant 0) and one-window-per-CTA (variant 8).
set -e
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in 0 8; do
  python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --variant $v > gpurun_out/plain_v$v.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:'dp_(pack|cta)_kernel' -s 2 -c 1 \
      -o gpurun_out/prof_c2_v$v -f python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline --variant $v \
      > gpurun_out/ncu_v$v.log 2>&1
done

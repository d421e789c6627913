#!/bin/bash
# A/B of the c2 DP kernels (variant 0 = automatic, 8 = one window per CTA) + ncu of the top kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_full.py -q -k "lockstep or c2" -x 2>&1 | tail -3
for v in 0 8; do python bench.py --workload c2 --steps 50 --warmup 5 --no-cpu-baseline --variant $v > gpurun_out/ab_c2_v$v.json 2>&1; done
python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_v0.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'dp_(pack|cta)_kernel' -s 2 -c 1 \
    -o gpurun_out/prof_c2_v0 -f python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_v0.log 2>&1

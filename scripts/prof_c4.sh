#!/bin/bash
# c4: bench (exchange on / off) and ncu --set full of the long-window DP kernel (exchange on / off)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_long.py -q -x 2>&1 | tail -2
python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c4.json 2>&1
TURBO_GRID_DEBUG=1 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_c4_noexch.json 2>&1
for x in 0 1; do
TURBO_GRID_DEBUG=$x python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c4_plain_$x.log 2>&1 && \
TURBO_GRID_DEBUG=$x ncu --set full --clock-control none --import-source on -k regex:'dp_grid_kernel' -s 1 -c 1 \
    -o gpurun_out/prof_c4_x$x -f python bench.py --workload c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c4_ncu_$x.log 2>&1
done

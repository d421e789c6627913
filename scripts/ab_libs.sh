#!/bin/bash
# A/B of library builds on the same box: bench WORKLOAD with each paper_2207_00172_b200/ab/*.so, 3 rounds
cd "${GRAFT_REPO_ROOT:-/root/repo}"
W=${1:-c4}
for r in 1 2 3; do
  for lib in paper_2207_00172_b200/ab/*.so; do
    n=$(basename $lib .so)
    TURBO_LIB=$lib python bench.py --workload $W --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${W}_${n}_$r.json 2>&1
  done
done

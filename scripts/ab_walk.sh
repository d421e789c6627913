#!/bin/bash
# same-box A/B of the fused smem walk: base, prefetched-cost walk (TURBO_WALK_PF), speculative walk (TURBO_DP_DEBUG=256)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for W in "$@"; do
for r in 1 2 3; do
  TURBO_LIB=paper_2207_00172_b200/ab/a_base.so python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/abw_${W}_base_$r.json 2>&1
  TURBO_LIB=paper_2207_00172_b200/ab/b_walkpf.so python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/abw_${W}_pf_$r.json 2>&1
  TURBO_DP_DEBUG=256 TURBO_LIB=paper_2207_00172_b200/ab/a_base.so python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/abw_${W}_spec_$r.json 2>&1
done
done

#!/bin/bash
# usage: scripts/sweep.sh "<workload>:<warps> ..."  -> gpurun_out/sweep.txt
out=gpurun_out/sweep.txt; : > $out
for spec in "$@"; do
  w=${spec%%:*}; g=${spec##*:}
  if [ "$g" = "auto" ]; then unset TURBO_DP_WARPS; else export TURBO_DP_WARPS=$g; fi
  r=$(timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu-baseline 2>&1 | tail -1)
  echo "$w G=$g $(echo "$r" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dp_ms %.4f frac %.3f step_ms %.4f' % (d['dp_ms'], d['roofline']['frac'], d['ms_per_step']))" 2>&1)" >> $out
done
unset TURBO_DP_WARPS

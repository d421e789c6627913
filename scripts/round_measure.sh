#!/bin/bash
# One measurement pass of the round (run under gpurun): bench lines for every workload, the
# reference arm, the ncu launch list of the default (c2) bench command, and ncu --set full of
# each workload's dominant DP kernel. Results land in gpurun_out/ (copied to profiles/ by
# scripts/collect_round.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/round
R=gpurun_out/round
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $R/gpu.txt 2>&1
for w in c2 c3 c5 c4 c1 lw; do
  python bench.py --workload $w --steps 20 --warmup 5 --cpu-seconds 8 > $R/bench_$w.json 2> $R/bench_$w.err
done
python bench.py --workload b2 --steps 20 --warmup 5 --cpu-seconds 5 > $R/bench_b2.json 2> $R/bench_b2.err
python bench.py --impl reference --workload c2 --steps 5 --warmup 1 > $R/bench_reference_c2.json 2> $R/bench_reference_c2.err
# launch list of the default bench command (cold-cache, serialised: compare shares)
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $R/plain_default.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $R/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $R/ncu_launches.log 2>&1
# ncu --set full of the dominant kernel per workload (after a plain run of the same command)
prof() {  # name workload kernel-regex skip
  python bench.py --workload $2 --steps 1 --warmup 3 --no-cpu-baseline > $R/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c 1 -o $R/$1 -f \
      python bench.py --workload $2 --steps 1 --warmup 3 --no-cpu-baseline > $R/ncu_$1.log 2>&1
}
prof full_schedule_c2 c2 'dp_cta_kernel' 2
prof full_schedule_c3 c3 'dp_cta_kernel' 2
prof full_grid_c4 c4 'dp_grid_kernel' 1
prof full_schedule_c5_cls3 c5 'dp_cta_kernel' 3
prof full_gen_c5_cls2 c5 'dp_gen_kernel' 3
prof full_batched_b2 b2 'batched_kernel' 2
prof full_cluster_lw lw 'dp_cluster_kernel' 1
# summaries on the box (only gpurun_out/ travels back, <= 64 MiB): JSON + CSV, then drop the reports
python scripts/collect_round.py ${TAG:-r02} $R/collected > $R/collect.log 2>&1
rm -f $R/*.ncu-rep
ls -la $R $R/collected

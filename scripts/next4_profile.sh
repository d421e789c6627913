python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/gpu_batched.log 2>&1
python bench.py --workload b2 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:batched_kernel -c 1 -o gpurun_out/prof_b2 python bench.py --workload b2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_b2.log 2>&1
python - <<'PY'
import csv, io, json, subprocess
out = subprocess.run(["ncu", "-i", "gpurun_out/prof_b2.ncu-rep", "--page", "raw", "--csv", "--metrics",
                      "smsp__inst_executed.sum,gpu__time_duration.sum"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
d = {"workload": "b2", "kernel": "turbo::batched_kernel", "warp_instructions_per_launch": float(v[h.index("smsp__inst_executed.sum")]),
     "ncu_duration": v[h.index("gpu__time_duration.sum")] + " " + rows[1][h.index("gpu__time_duration.sum")],
     "source": "profiles/r01_ncu_full_batched_b2_summary.json (ncu --set full, one launch)"}
json.dump(d, open("profiles/issue_b2.json", "w"), indent=1)
json.dump(d, open("gpurun_out/issue_b2.json", "w"), indent=1)
PY
python bench.py --workload b2 > gpurun_out/bench_b2.log 2>&1
python bench.py --workload b2 --impl reference --steps 5 > gpurun_out/bench_b2_ref.log 2>&1

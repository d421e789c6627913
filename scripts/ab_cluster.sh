cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2; do for lib in paper_2207_00172_b200/ab/*.so; do n=$(basename $lib .so); TURBO_LIB=$lib python scripts/cluster_vs_grid.py 64 300 6 60000 > gpurun_out/abcl_${n}_a$r.json 2>&1; TURBO_LIB=$lib python scripts/cluster_vs_grid.py 148 300 8 30000 > gpurun_out/abcl_${n}_b$r.json 2>&1; done; done

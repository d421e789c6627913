#!/bin/bash
# ncu --set full + SASS source page of the cluster kernel on a batch of long windows
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/src
ncu --set full --clock-control none --import-source on -k regex:dp_cluster_kernel -s 1 -c 1 -o gpurun_out/src/cluster -f \
    python scripts/cluster_vs_grid.py ${1:-64} ${2:-100} ${3:-6} ${4:-60000} > gpurun_out/src/ncu_cluster.log 2>&1
ncu -i gpurun_out/src/cluster.ncu-rep --page raw --csv > gpurun_out/src/raw_cluster.csv 2>&1
ncu -i gpurun_out/src/cluster.ncu-rep --page source --csv --print-source sass > gpurun_out/src/sass_cluster.csv 2>&1
ncu -i gpurun_out/src/cluster.ncu-rep --page details --csv > gpurun_out/src/details_cluster.csv 2>&1
rm -f gpurun_out/src/cluster.ncu-rep

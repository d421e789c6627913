#!/bin/bash
# Build an A/B variant of libturbo.so: scripts/build_ab.sh NAME "-DFLAG ..." -> paper_2207_00172_b200/ab/NAME.so
# (objects under /tmp/turbo_ab_NAME; bench with TURBO_LIB=... or scripts/ab_libs.sh)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
DEFS="$*"
OBJ=/tmp/turbo_ab_$NAME
mkdir -p $OBJ paper_2207_00172_b200/ab
pids=()
for s in paper_2207_00172_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr $DEFS -I include -I paper_2207_00172_b200/csrc -c -o $OBJ/$(basename $s .cu).o $s &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o paper_2207_00172_b200/ab/$NAME.so $OBJ/*.o
echo built paper_2207_00172_b200/ab/$NAME.so

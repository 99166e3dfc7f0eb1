#!/bin/bash
# Sweep-kernel tuning: threads per block x target parts (warps per row), per workload.
TAG=${1:-tune}
for w in ${WORKLOADS:-c3a_27pt_128_ilu1 c3b_27pt_128_ilu2}; do
  for cfg in ${CFGS:-"128 1" "128 2" "128 4" "256 2" "256 4" "256 8"}; do
    set -- $cfg
    export FASTILU_TSELL_THREADS=$1 FASTILU_TSELL_PARTS=$2
    echo "== $w threads=$1 parts=$2"
    timeout 200 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1
  done
done > gpurun_out/${TAG}_tune.log 2>&1

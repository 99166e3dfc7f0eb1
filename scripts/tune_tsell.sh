#!/bin/bash
# Sweep-kernel tuning: threads per block x target parts (warps per row), per workload.
TAG=${1:-tune}
CFG_LIST=${CFGS:-"128:1 128:2 128:4 256:2 256:4 256:8"}
for w in ${WORKLOADS:-c3a_27pt_128_ilu1 c3b_27pt_128_ilu2}; do
  for cfg in $CFG_LIST; do
    th=${cfg%%:*}; pa=${cfg##*:}
    export FASTILU_TSELL_THREADS=$th FASTILU_TSELL_PARTS=$pa
    echo "== $w threads=$th parts=$pa"
    timeout 300 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1
  done
done > gpurun_out/${TAG}_tune.log 2>&1

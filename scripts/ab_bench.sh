#!/bin/bash
# A/B bench of env settings: ab_bench.sh TAG "ENV1" "ENV2" ... over $WORKLOADS
TAG=$1; shift
for w in ${WORKLOADS:-c3a_27pt_128_ilu1 c3b_27pt_128_ilu2 c4_27pt_256_ilu1}; do
  for e in "$@"; do
    echo "== $w $e"
    env $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1
  done
done > gpurun_out/${TAG}_tune.log 2>&1

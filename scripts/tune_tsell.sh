#!/bin/bash
# Sweep-kernel tuning: accumulator chunk (registers) x threads per block, per workload.
TAG=${1:-tune}
for w in c3a_27pt_128_ilu1 c3b_27pt_128_ilu2; do
  for th in 128 256; do
    for ch in 0 40 32 20; do
      if [ "$ch" = "0" ]; then unset FASTILU_TSELL_CHUNK; else export FASTILU_TSELL_CHUNK=$ch; fi
      export FASTILU_TSELL_THREADS=$th
      echo "== $w threads=$th chunk=$ch"
      timeout 200 python bench.py --workload $w --steps 5 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1
    done
  done
done > gpurun_out/${TAG}_tune.log 2>&1

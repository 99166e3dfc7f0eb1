#!/bin/bash
# quick check of the staged sweep: debug JIT log, parity subset, A/B bench
TAG=${1:-st}
FASTILU_DEBUG=1 timeout 300 python bench.py --workload c3a_27pt_128_ilu1 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_dbg.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/${TAG}_parity.log 2>&1
WORKLOADS="c3a_27pt_128_ilu1 c3b_27pt_128_ilu2 c4_27pt_256_ilu1" bash scripts/ab_bench.sh ${TAG} FASTILU_TSELL_STAGED=0 FASTILU_TSELL_STAGED=1

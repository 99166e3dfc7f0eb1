#!/bin/bash
# usage: bash scripts_gpu_run.sh TAG  -- runs gpu tests + benches, writes gpurun_out/TAG_*.log
TAG=${1:-run}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/${TAG}_gputest.log
for w in c2_7pt_128_ilu0 c3a_27pt_128_ilu1 c3b_27pt_128_ilu2; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e; done > gpurun_out/${TAG}_bench_small.log 2>&1
timeout 500 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_bench256.log 2>&1

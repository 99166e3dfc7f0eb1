#!/bin/bash
# sweep 1 with its own block shape: parity (variants, compute_host pipeline, multi-rank) + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r1k_tests.log
for r in 1 2; do timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r1k_bench$r.log 2>&1; done
timeout 300 python bench.py --workload c3a_27pt_128_ilu1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r1k_c3a.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r1i_smi.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r1i_tests.log
for r in 1 2; do timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r1i_bench$r.log 2>&1; done

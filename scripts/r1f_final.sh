#!/bin/bash
# round-1 final check: GPU tests, smoke, default bench, config-3 sweeps to convergence, c2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r1g_gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1g_smoke.log 2>&1
timeout 500 python bench.py > gpurun_out/r1g_bench.log 2>&1
for w in c3a_27pt_128_ilu1 c3b_27pt_128_ilu2; do
  timeout 300 python bench.py --workload $w --tol 1e-10 --steps 5 --warmup 3 > gpurun_out/r1g_tol_$w.log 2>&1
done
timeout 300 python bench.py --workload c2_7pt_128_ilu0 --steps 10 --warmup 3 > gpurun_out/r1g_c2.log 2>&1

#!/bin/bash
# round-1 final: every GPU test, smoke, default bench, reference arm, c3 to convergence
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r1n_gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1n_smoke.log 2>&1
timeout 500 python bench.py > gpurun_out/r1n_bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1n_ref.log 2>&1
for w in c3a_27pt_128_ilu1 c3b_27pt_128_ilu2; do
  timeout 300 python bench.py --workload $w --tol 1e-10 --steps 5 --warmup 3 > gpurun_out/r1n_tol_$w.log 2>&1
done

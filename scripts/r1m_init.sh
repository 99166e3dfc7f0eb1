#!/bin/bash
# A/B: c4 sweep 1 tile rows and ring depth
mkdir -p gpurun_out
for w in c4_27pt_256_ilu1; do
  for e in "X=0" "FASTILU_TSELL_INIT_THREADS=384" "FASTILU_TSELL_STAGES_INIT=3" "FASTILU_TSELL_STAGES_INIT=4" "FASTILU_TSELL_INIT_THREADS=384 FASTILU_TSELL_STAGES_INIT=3" "FASTILU_TSELL_INIT_THREADS=288"; do
    echo "== $w $e"
    env FASTILU_DEBUG=1 $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "^\{|rror" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/step %.3f sweep1 %.3f launch %.3f apply %.3f frac %.3f %s'%(d['ms_per_step'],d['sweep1_ms'],d['sweep_launch_ms'],d['apply_ms'],d['roofline']['frac'], d['kernel_config'][-40:]))
    else: print(l.strip()[:200])"
  done
done > gpurun_out/r1m_init.log 2>&1
timeout 300 python bench.py --workload c3b_27pt_128_ilu2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r1m_c3b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "variants or first_sweep or compute_host or stencils or convergence" 2>&1 | tail -3 > gpurun_out/r1m_tests.log

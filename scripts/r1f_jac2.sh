#!/bin/bash
# paired Jacobi sweeps: parity of every variant, then A/B of lag / occupancy at c4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r1f_jac2_parity.log
for w in c4_27pt_256_ilu1; do
  for e in "FASTILU_JAC2=0" "X=0" "FASTILU_JAC2_LAG=600" "FASTILU_JAC2_LAG=900" "FASTILU_JAC2_LAG=1800" "FASTILU_JAC2_BPS=4 FASTILU_JAC2_LAG=650" "FASTILU_JAC2_BPS=4 FASTILU_JAC2_LAG=400" "FASTILU_JAC2_BPS=6 FASTILU_JAC2_LAG=950"; do
    echo "== $w $e"
    env $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "^\{|Error|error" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/step %.3f sweep1 %.3f launch %.3f apply %.3f frac %.3f'%(d['ms_per_step'],d['sweep1_ms'],d['sweep_launch_ms'],d['apply_ms'],d['roofline']['frac']))
    else: print(l.strip())"
  done
done > gpurun_out/r1f_jac2.log 2>&1

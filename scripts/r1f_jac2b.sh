#!/bin/bash
mkdir -p gpurun_out
for m in 1 3; do FASTILU_JAC2_MODE=$m timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "variants and (paired or streaming)" 2>&1 | tail -2; done > gpurun_out/r1f_jac2b_parity.log
for w in c4_27pt_256_ilu1; do
  for e in "FASTILU_JAC2=0" "FASTILU_JAC2_MODE=1" "FASTILU_JAC2_MODE=2" "FASTILU_JAC2_MODE=3" "FASTILU_JAC2_MODE=3 FASTILU_JAC2_LAG=700" "FASTILU_JAC2_MODE=3 FASTILU_JAC2_LAG=1800" "FASTILU_JAC2_MODE=1 FASTILU_JAC2_LAG=3000"; do
    echo "== $w $e"
    env $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "^\{|Error|error" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/step %.3f sweep1 %.3f launch %.3f apply %.3f frac %.3f'%(d['ms_per_step'],d['sweep1_ms'],d['sweep_launch_ms'],d['apply_ms'],d['roofline']['frac']))
    else: print(l.strip())"
  done
done > gpurun_out/r1f_jac2b.log 2>&1

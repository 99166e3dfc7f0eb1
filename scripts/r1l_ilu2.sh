#!/bin/bash
# A/B: ILU(2) init-fused sweep 1 block shape
mkdir -p gpurun_out
for w in c3b_27pt_128_ilu2; do
  for e in "X=0" "FASTILU_TSELL_INIT_PARTS=2 FASTILU_TSELL_INIT_THREADS=512" "FASTILU_TSELL_INIT_PARTS=2 FASTILU_TSELL_INIT_THREADS=256" "FASTILU_TSELL_INIT_PARTS=1 FASTILU_TSELL_INIT_THREADS=256" "FASTILU_TSELL_INIT_PARTS=3 FASTILU_TSELL_INIT_THREADS=576"; do
    echo "== $w $e"
    env FASTILU_DEBUG=1 $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "^\{|rror" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/step %.3f sweep1 %.3f launch %.3f apply %.3f frac %.3f %s'%(d['ms_per_step'],d['sweep1_ms'],d['sweep_launch_ms'],d['apply_ms'],d['roofline']['frac'], d['kernel_config'][-40:]))
    else: print(l.strip()[:200])"
  done
done > gpurun_out/r1l_ilu2.log 2>&1

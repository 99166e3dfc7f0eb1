#!/bin/bash
# repeated A/B: full sweep with 1 vs 2 part-warps per slice (256-row tiles)
mkdir -p gpurun_out
for rep in 1 2 3; do
for w in c4_27pt_256_ilu1 c3a_27pt_128_ilu1; do
  for e in "X=0" "FASTILU_TSELL_ST_PARTS=1 FASTILU_TSELL_ST_THREADS=256"; do
    echo "== $rep $w $e"
    env $e timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "^\{|rror" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/step %.3f sweep1 %.3f launch %.3f apply %.3f mhz %s'%(d['ms_per_step'],d['sweep1_ms'],d['sweep_launch_ms'],d['apply_ms'],d['clocks']['sm_mhz']))
    else: print(l.strip()[:200])"
  done
done
done > gpurun_out/r1p_parts.log 2>&1

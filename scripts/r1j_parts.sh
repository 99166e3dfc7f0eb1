#!/bin/bash
# A/B: one part-warp per slice (all targets of a row in one thread) with 256-320-row tiles
mkdir -p gpurun_out
for w in c4_27pt_256_ilu1 c3a_27pt_128_ilu1; do
  for e in "X=0" "FASTILU_TSELL_ST_PARTS=1 FASTILU_TSELL_ST_THREADS=256" "FASTILU_TSELL_ST_PARTS=1 FASTILU_TSELL_ST_THREADS=288" "FASTILU_TSELL_ST_PARTS=1 FASTILU_TSELL_ST_THREADS=320" "FASTILU_TSELL_ST_PARTS=1 FASTILU_TSELL_ST_THREADS=320 FASTILU_TSELL_ST_MINB=1"; do
    echo "== $w $e"
    env FASTILU_DEBUG=1 $e timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "staged|^\{|rror" | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms/step %.3f sweep1 %.3f launch %.3f apply %.3f frac %.3f'%(d['ms_per_step'],d['sweep1_ms'],d['sweep_launch_ms'],d['apply_ms'],d['roofline']['frac']))
    else: print(l.strip()[:200])"
  done
done > gpurun_out/r1j_parts2.log 2>&1

#!/bin/bash
# round-1 final evidence: launch list of one c4 step and one --set full capture of it
mkdir -p gpurun_out
W=c4_27pt_256_ilu1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r1i_launches.csv python scripts/profile_step.py --workload $W > gpurun_out/r1i_ncu_list.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:fastilu -c 12 \
  -o gpurun_out/r1i_full python scripts/profile_step.py --workload $W > gpurun_out/r1i_ncu_full.log 2>&1
ls -la gpurun_out/ >> gpurun_out/r1i_ncu_full.log

#!/bin/bash
# final launch list + full capture of the step (sweep 1 with its own block shape)
mkdir -p gpurun_out
W=c4_27pt_256_ilu1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r1o_launches.csv python scripts/profile_step.py --workload $W > gpurun_out/r1o_ncu_list.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:fastilu -c 12 \
  -o gpurun_out/r1o_full python scripts/profile_step.py --workload $W > gpurun_out/r1o_ncu_full.log 2>&1

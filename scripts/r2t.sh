# round-2 t: timing probe of a fused multiply-subtract per term (NOT the oracle's rounding)
AB_ENVS="FASTILU_DEFAULT=1;FASTILU_TSELL_ST_OPTS=34560 FASTILU_TSELL_INIT_OPTS=38656;FASTILU_DEFAULT=1;FASTILU_TSELL_ST_OPTS=34560 FASTILU_TSELL_INIT_OPTS=38656" WORKLOADS="c3a_27pt_128_ilu1 c4_27pt_256_ilu1" bash scripts/gpu_session.sh r2t ab

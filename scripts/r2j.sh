# round-2 j: column-major boxes / no presence select / 640-thread tiles -- parity variants, A/B
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "variants" 2>&1 | tail -4 > gpurun_out/r2j_tests.log
AB_ENVS="FASTILU_TSELL_ST_OPTS=1792;FASTILU_TSELL_ST_OPTS=5888;FASTILU_TSELL_ST_OPTS=14080;FASTILU_TSELL_ST_OPTS=9984;FASTILU_TSELL_ST_OPTS=14080 FASTILU_TSELL_ST_THREADS=640;FASTILU_TSELL_ST_OPTS=1792 FASTILU_TSELL_ST_THREADS=640 FASTILU_DEBUG=1;FASTILU_TSELL_ST_OPTS=14080 FASTILU_DEBUG=1" bash scripts/gpu_session.sh r2j ab

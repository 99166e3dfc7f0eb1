# round-2 k: per-template staged defaults (ILU(2): 640 threads, column-major, no select; init
# sweep column-major) -- full GPU tests, c3b option A/B at 640 threads, default bench lines
bash scripts/gpu_session.sh r2k tests
AB_ENVS="FASTILU_TSELL_ST_OPTS=14080 FASTILU_TSELL_ST_THREADS=640;FASTILU_TSELL_ST_OPTS=9984 FASTILU_TSELL_ST_THREADS=640;FASTILU_TSELL_ST_OPTS=5888 FASTILU_TSELL_ST_THREADS=640;FASTILU_TSELL_ST_OPTS=1792 FASTILU_TSELL_ST_THREADS=512;FASTILU_DEFAULT=1" WORKLOADS="c3b_27pt_128_ilu2" bash scripts/gpu_session.sh r2k ab
bash scripts/gpu_session.sh r2k small bench

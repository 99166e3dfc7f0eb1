# round-2 A/B: column-split ring vs the one-box ring; solve_host pipeline; parity subsets
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "split or solve_host or variants" 2>&1 | tail -4 > gpurun_out/r2f_tests.log
AB_ENVS="FASTILU_TSELL_SPLIT=0;FASTILU_TSELL_SPLIT=1;FASTILU_TSELL_SPLIT=1 FASTILU_TSELL_STAGES=3;FASTILU_TSELL_SPLIT=0" bash scripts/gpu_session.sh r2f ab
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2f_bench_pipe.log 2>&1
FASTILU_NO_SOLVE_PIPELINE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2f_bench_nopipe.log 2>&1

# round-2 q: template SpMV for GMRES + unroll-4 orthogonalisation -- GMRES tests, launch list,
# config-5 bench
timeout 1200 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_multirank.py -q -x -k "gmres or set_factors" 2>&1 | tail -4 > gpurun_out/r2q_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2q_gmres_launches.csv python scripts/profile_gmres.py --iters 60 > gpurun_out/r2q_gmres.log 2>&1
timeout 1500 python bench.py --workload c5_aniso7pt_256_ilu0 --steps 5 --warmup 3 > gpurun_out/r2q_c5.log 2>&1

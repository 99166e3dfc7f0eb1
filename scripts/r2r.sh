# round-2 r: GMRES with selective reorthogonalisation -- tests, launch list, config-5 bench
timeout 1200 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_multirank.py -q -x -k "gmres or set_factors" 2>&1 | tail -4 > gpurun_out/r2r_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2r_gmres_launches.csv python scripts/profile_gmres.py --iters 60 > gpurun_out/r2r_gmres.log 2>&1
timeout 1500 python bench.py --workload c5_aniso7pt_256_ilu0 --steps 5 --warmup 3 > gpurun_out/r2r_c5.log 2>&1
FASTILU_GMRES_CGS2=1 timeout 1500 python bench.py --workload c5_aniso7pt_256_ilu0 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2r_c5_cgs2.log 2>&1

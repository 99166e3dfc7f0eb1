# round-2 o: GMRES orthogonalisation kernels (one pass per V_j, norm fused, one sync per
# iteration on one GPU) -- GMRES tests, config-5 bench
timeout 1200 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_multirank.py -q -x -k "gmres or set_factors" 2>&1 | tail -4 > gpurun_out/r2o_tests.log
bash scripts/gpu_session.sh r2o c5

# round-2 p: GMRES kernel launch list (one restart cycle of 60 iterations at 256^3)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r2p_gmres_launches.csv python scripts/profile_gmres.py --iters 60 > gpurun_out/r2p_gmres.log 2>&1

# round-2 s: final-state evidence -- GPU tests + smoke, default bench + reference arm, small
# configs, config 3 to convergence, config 5 arms, c4 launch list, ncu --set full of one c4 step
bash scripts/gpu_session.sh r2s tests bench small tol c5 launches full

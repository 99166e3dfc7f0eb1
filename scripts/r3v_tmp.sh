set -u
mkdir -p gpurun_out
FASTILU_TRACE=1 timeout 600 python scripts/e2e_trace.py --reps 3 > gpurun_out/r3v_trace.log 2>&1
FASTILU_SOLVE_NOPIPE=1 FASTILU_TRACE=1 timeout 600 python scripts/e2e_trace.py --reps 2 > gpurun_out/r3v_trace_nopipe.log 2>&1
timeout 600 python scripts/h2d_probe.py > gpurun_out/r3v_h2d.log 2>&1
nvidia-smi topo -m > gpurun_out/r3v_topo.log 2>&1; nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" >> gpurun_out/r3v_topo.log 2>&1

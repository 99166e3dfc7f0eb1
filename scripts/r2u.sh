# round-2 u: compute-sanitizer over the final kernels (column-major init / ILU(2) staged sweeps,
# template SpMV and the new GMRES orthogonalisation kernels included)
timeout 600 python tests/sanitize_case.py > gpurun_out/r2u_plain.log 2>&1
bash scripts/gpu_session.sh r2u sanitize

# round-2 i: final-code evidence -- sanitizer over every default-path kernel (extended case),
# ncu --set full of one c4 step
timeout 600 python tests/sanitize_case.py > gpurun_out/r2i_plain.log 2>&1
bash scripts/gpu_session.sh r2i sanitize full

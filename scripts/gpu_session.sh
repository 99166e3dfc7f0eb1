#!/usr/bin/env bash
# One parametrised runner for the GPU box (replaces round 1's one-off r1*_*.sh launchers).
#   bash scripts/gpu_session.sh TAG STEP [STEP ...]
# Every step writes gpurun_out/TAG_<step>.log (JSON lines for the benches).  Steps:
#   tests      pytest -m gpu (all GPU tests) + smoke()
#   bench      default bench.py line (c4) + the reference arm
#   small      bench lines of c2, c3a, c3b (no e2e / cpu leg)
#   tol        config 3 "to convergence" (c3a, c3b at tol 1e-10)
#   c5         config 5 GMRES arms (bench.py --workload c5_aniso7pt_256_ilu0)
#   launches   ncu launch list of one c4 step (per-kernel times)          -> TAG_launches.csv
#   full       ncu --set full of the step's kernels (-c $NCU_COUNT)       -> TAG_full.ncu-rep
#   sanitize   compute-sanitizer memcheck/racecheck/synccheck/initcheck on a small ragged grid
#   ab         A/B of env settings: AB_ENVS="A=1 B=2;A=0" over $WORKLOADS (each log line is
#              preceded by "== workload env"; the round-2 A/B logs under profiles/ keep them)
#   variants   the template-kernel variant parity tests only (bitwise vs the oracle)
#   gmres      ncu launch list (time + DRAM bytes) of one GMRES(60) cycle on config 5
#   gmrestest  the GMRES GPU tests only (single GPU, in-process ranks, async) + config 5 (no arm C)
set -u
TAG=$1; shift
mkdir -p gpurun_out
W4=${WORKLOAD:-c4_27pt_256_ilu1}
for step in "$@"; do
  case $step in
    tests)
      timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${TAG}_tests.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" \
        > gpurun_out/${TAG}_smoke.log 2>&1 ;;
    bench)
      timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
      timeout 400 python bench.py --impl reference --steps 3 --warmup 3 >> gpurun_out/${TAG}_bench.log 2>&1 ;;
    small)
      for w in c2_7pt_128_ilu0 c3a_27pt_128_ilu1 c3b_27pt_128_ilu2; do
        timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e
      done > gpurun_out/${TAG}_small.log 2>&1 ;;
    tol)
      for w in c3a_27pt_128_ilu1 c3b_27pt_128_ilu2; do
        timeout 300 python bench.py --workload $w --tol 1e-10 --steps 5 --warmup 3 --no-e2e
      done > gpurun_out/${TAG}_tol.log 2>&1 ;;
    c5)
      timeout 1500 python bench.py --workload c5_aniso7pt_256_ilu0 --steps 5 --warmup 3 --arm-c \
        > gpurun_out/${TAG}_c5.log 2>&1 ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_step.py --workload $W4 \
        > gpurun_out/${TAG}_launches.log 2>&1 ;;
    full)
      timeout 1800 ncu --set full --clock-control none --import-source on -k regex:fastilu \
        -c ${NCU_COUNT:-12} -o gpurun_out/${TAG}_full python scripts/profile_step.py --workload $W4 \
        > gpurun_out/${TAG}_full.log 2>&1 ;;
    sanitize)
      for tool in memcheck racecheck synccheck initcheck; do
        echo "== $tool"
        timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/sanitize_case.py 2>&1 | tail -25
      done > gpurun_out/${TAG}_sanitize.log 2>&1 ;;
    variants)
      timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "variants" 2>&1 | tail -4 \
        > gpurun_out/${TAG}_variants.log ;;
    gmres)
      timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/${TAG}_gmres_launches.csv \
        python scripts/profile_gmres.py --iters 60 > gpurun_out/${TAG}_gmres.log 2>&1 ;;
    gmrestest)
      timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_multirank.py \
        tests/test_gpu_async.py -q -x -k "gmres or dcgs2 or restarts or set_factors" 2>&1 | tail -6 \
        > gpurun_out/${TAG}_gmrestest.log
      timeout 900 python bench.py --workload c5_aniso7pt_256_ilu0 --steps 3 --warmup 3 --no-cpu \
        > gpurun_out/${TAG}_c5.log 2>&1 ;;
    ab)
      IFS=';' read -ra envs <<< "${AB_ENVS:-}"
      for w in ${WORKLOADS:-c3a_27pt_128_ilu1 c3b_27pt_128_ilu2 c4_27pt_256_ilu1}; do
        for e in "${envs[@]}"; do
          echo "== $w $e"
          env $e timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1
        done
      done > gpurun_out/${TAG}_ab.log 2>&1 ;;
    *) echo "unknown step $step" >&2 ;;
  esac
done

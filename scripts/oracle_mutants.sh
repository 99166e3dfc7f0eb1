#!/usr/bin/env bash
# Mutation check of the oracle pins (VERDICT r1 "next round" item 1): each mutant below must make
# at least one `-m "not gpu"` oracle test fail.  Runs on a scratch copy; the repo is untouched.
#   1. swapped damping weights in the sweep  (w old + (1-w) new instead of (1-w) old + w new)
#   2. swapped damping weights in the Jacobi lower sweep
#   3. a misplaced warm-up embedding          (one S_{L-1} value dropped to 0 inside S_L)
#   4. a left-to-right residual sum           (instead of the exactly rounded one)
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
W="$(mktemp -d)"
trap 'rm -rf "$W"' EXIT
run() {  # $1 = label; the mutated tree is in $W
  rm -rf "$W/oracle/build"
  if (cd "$W" && timeout 600 python -m pytest tests/test_oracle_numeric.py -q -p no:cacheprovider \
        > "$W/log" 2>&1); then
    echo "MUTANT SURVIVED: $1"; return 1
  fi
  echo "killed: $1 ($(grep -c '^FAILED' "$W/log") failing tests)"
}
fresh() { rm -rf "$W"/*; cp -r "$ROOT/oracle" "$ROOT/problems" "$ROOT/tests" "$ROOT/pytest.ini" "$W/"; }
ok=0
fresh; sed -i 's/(1.0 - omega) \* old\[p\] + omega \* l;/omega * old[p] + (1.0 - omega) * l;/; s/(1.0 - omega) \* old\[p\] + omega \* acc;/omega * old[p] + (1.0 - omega) * acc;/' "$W/oracle/fastilu_oracle.c"
run "sweep damping weights swapped" || ok=1
fresh; sed -i 's/(1.0 - omega) \* zo\[i\] + omega \* acc;/omega * zo[i] + (1.0 - omega) * acc;/' "$W/oracle/fastilu_oracle.c"
run "Jacobi damping weights swapped" || ok=1
fresh; sed -i 's/            vals\[pos\] = pvals/            vals[pos] = pvals; vals[pos[-1]] = 0.0/' "$W/oracle/__init__.py"
run "warm-up embedding drops an entry" || ok=1
fresh; sed -i 's/  \*resid = sqrt(orc_fsum_result(&total));/  { double t = 0.0; for (int j = 0; j < total.n; j++) t += total.p[j]; *resid = sqrt(t) * (1.0 + 4e-16); }/' "$W/oracle/fastilu_oracle.c"
run "residual not exactly rounded" || ok=1
exit $ok

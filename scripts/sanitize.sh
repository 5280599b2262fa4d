#!/usr/bin/env bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over every sweep-kernel path at
# small sizes; each case is also a bit-exact parity check against the oracle.
# Usage (on the GPU box): bash scripts/sanitize.sh TAG
TAG=${1:-san}; OUT=gpurun_out/$TAG; mkdir -p $OUT
S="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() {  # tool case [env]
  local tool=$1 c=$2; shift 2
  env "$@" timeout 900 $S --tool $tool python scripts/sanitize_cases.py $c > $OUT/${tool}_$c.txt 2>&1
  echo "$tool $c exit $?" | tee -a $OUT/summary.txt
}
timeout 600 python scripts/sanitize_cases.py > $OUT/plain.txt 2>&1; echo "plain exit $?" | tee -a $OUT/summary.txt
for tool in racecheck memcheck synccheck initcheck; do
  run $tool kpz_full
  run $tool kpz_general
  run $tool kpz_small
  run $tool kpz_sub1
  run $tool kpz_sub8
  run $tool kpz_sharded
  run $tool kmc_wide
  run $tool kmc_wide1 LFG_KMC_PC=0
  run $tool kmc_narrow LFG_KMC_WIDE=0
  run $tool kmc_quad
  run $tool kmc_32
done
run memcheck kpz_tensor
run initcheck kpz_tensor

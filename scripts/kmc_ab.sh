#!/usr/bin/env bash
# KMC A/B: default library vs variants under _lib/variants (kmc_bench at L = 256, 512).
TAG=${1:-kmcab}; OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "$TESTS" ] && timeout 900 python -m pytest $TESTS -x -q -m gpu > $OUT/pytest.txt 2>&1
for L in ${SIZES:-256}; do
  timeout 200 python scripts/kmc_bench.py $L 30 > $OUT/main_$L.txt 2>&1
  for v in paper_1204_5072_b200/_lib/variants/*/liblfg.so; do
    n=$(basename $(dirname $v))
    LFG_LIB=$PWD/$v timeout 200 python scripts/kmc_bench.py $L 30 > $OUT/${n}_$L.txt 2>&1
    [ -n "$VTESTS" ] && LFG_LIB=$PWD/$v timeout 300 python -m pytest $VTESTS -x -q -m gpu > $OUT/pytest_$n.txt 2>&1
  done
done

#!/usr/bin/env bash
# KMC A/B, alternating arms 3x: default library vs every variant under _lib/variants
# (scripts/kmc_bench.py, 16^3 blocks, both active modes).
# Usage: bash scripts/kmc_ab3.sh TAG   (SIZES="256 512", default 256)
TAG=${1:-kmcab3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for i in 1 2 3; do
  for L in ${SIZES:-256}; do
    timeout 200 python scripts/kmc_bench.py $L 30 2>&1 | head -2 > $OUT/main_${L}_$i.txt
    for v in paper_1204_5072_b200/_lib/variants/*/liblfg.so; do
      [ -f "$v" ] || continue
      n=$(basename $(dirname $v))
      LFG_LIB=$PWD/$v timeout 200 python scripts/kmc_bench.py $L 30 2>&1 | head -2 > $OUT/${n}_${L}_$i.txt
    done
  done
done
for f in $OUT/*.txt; do
  echo $(basename $f) $(python -c "
import json
print(' '.join(str(round(json.loads(l)['att_per_ns'], 2)) for l in open('$f') if l.startswith('{')))")
done > $OUT/summary.txt

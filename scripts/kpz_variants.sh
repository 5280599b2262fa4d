#!/usr/bin/env bash
# Time the KPZ phase kernel for each library variant under paper_1204_5072_b200/_lib/variants/.
TAG=${1:-var}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in paper_1204_5072_b200/_lib/variants/*/liblfg.so; do
  n=$(basename $(dirname $v))
  LFG_LIB=$PWD/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_$n.json 2> $OUT/bench_$n.err
done

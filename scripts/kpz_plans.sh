#!/usr/bin/env bash
# Time the KPZ phase kernel for several DT block plans and library variants.
# Usage: bash scripts/kpz_plans.sh TAG "bx:by ..." [variant ...]
TAG=${1:-plans}; PLANS=${2:-"1024:128 1024:64 1024:32"}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
VARS=${@:-main}
for v in $VARS; do
  for p in $PLANS; do
    bx=${p%%:*}; by=${p##*:}
    if [ "$v" = main ]; then unset LFG_LIB; else export LFG_LIB=$PWD/paper_1204_5072_b200/_lib/variants/$v/liblfg.so; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc --block-x $bx --block-y $by \
        > $OUT/bench_${v}_${bx}x${by}.json 2> $OUT/bench_${v}_${bx}x${by}.err
  done
done

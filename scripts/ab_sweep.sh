#!/usr/bin/env bash
# A/B of the whole-sweep kernel vs four phase launches (and an optional old library variant).
TAG=${1:-ab}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/ -x -q -m gpu > $OUT/pytest.txt 2>&1
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc"
for i in 1 2; do
  timeout 300 $B > $OUT/bench_sweep_$i.json 2> $OUT/bench_sweep_$i.err
  LFG_KPZ_PHASE_LAUNCHES=1 timeout 300 $B > $OUT/bench_phase_$i.json 2> $OUT/bench_phase_$i.err
  for v in paper_1204_5072_b200/_lib/variants/*/liblfg.so; do
    n=$(basename $(dirname $v))
    LFG_LIB=$PWD/$v timeout 300 $B > $OUT/bench_${n}_$i.json 2> $OUT/bench_${n}_$i.err
  done
done

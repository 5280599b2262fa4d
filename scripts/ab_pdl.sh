#!/usr/bin/env bash
# A/B of chained (PDL + per-block flags) phase launches vs plain stream-ordered phases
# (and any library variants under paper_1204_5072_b200/_lib/variants/).
TAG=${1:-pdl}; OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "$SKIP_TESTS" ] || timeout 600 python -m pytest tests/test_kpz_gpu.py tests/test_shard_gpu.py tests/test_writelog_gpu.py -x -q -m gpu > $OUT/pytest.txt 2>&1
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc"
for i in 1 2 3; do
  timeout 300 $B > $OUT/bench_pdl_$i.json 2> $OUT/bench_pdl_$i.err
  LFG_KPZ_PDL=0 timeout 300 $B > $OUT/bench_nopdl_$i.json 2> $OUT/bench_nopdl_$i.err
  for v in paper_1204_5072_b200/_lib/variants/*/liblfg.so; do
    n=$(basename $(dirname $v))
    LFG_LIB=$PWD/$v timeout 300 $B > $OUT/bench_${n}_$i.json 2> $OUT/bench_${n}_$i.err
  done
done

#!/usr/bin/env bash
# A/B of KPZ bench arms selected by environment: ab_env.sh TAG "NAME=ENV ..." ...
# e.g. scripts/ab_env.sh s1 "pdl=" "plain=LFG_KPZ_PDL=0"
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "$TESTS" ] && timeout 900 python -m pytest $TESTS -x -q -m gpu > $OUT/pytest.txt 2>&1
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc"
for i in 1 2 3; do
  for arm in "$@"; do
    n=${arm%%=*}; e=${arm#*=}
    env $e timeout 300 $B > $OUT/bench_${n}_$i.json 2> $OUT/bench_${n}_$i.err
  done
done
for f in $OUT/bench_*.json; do
  echo $f $(python -c "import json;d=json.load(open('$f'));print(round(d['value'],1))" 2>&1 | tail -1)
done > $OUT/summary.txt

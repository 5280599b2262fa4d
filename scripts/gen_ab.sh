#!/usr/bin/env bash
# p < 1 (BASELINE C3 parameters) KPZ bench: default library vs variants.
TAG=${1:-gen}; OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "$TESTS" ] && timeout 900 python -m pytest $TESTS -x -q -m gpu > $OUT/pytest.txt 2>&1
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc --p 0.95 --q 0.05"
for i in 1 2; do
  timeout 300 $B > $OUT/main_$i.json 2>/dev/null
  for v in paper_1204_5072_b200/_lib/variants/*/liblfg.so; do
    [ -f "$v" ] || continue
    n=$(basename $(dirname $v))
    LFG_LIB=$PWD/$v timeout 300 $B > $OUT/${n}_$i.json 2>/dev/null
  done
done
for f in $OUT/*.json; do echo $f $(python -c "import json;print(round(json.load(open('$f'))['value'],1))" 2>&1 | tail -1); done > $OUT/summary.txt

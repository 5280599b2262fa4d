#!/usr/bin/env bash
# A/B of the KPZ bench: default library vs library variants (paper_1204_5072_b200/_lib/variants/NAME/liblfg.so),
# at p=1 (configs[1]) and p=0.95 q=0.05 (configs[2] parameters), alternating arms, 3 repetitions.
# Usage: bash scripts/ab_lib.sh TAG NAME...   (TESTS="tests/x.py" also runs those GPU tests on each variant)
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for n in "$@"; do
  [ -n "$TESTS" ] && LFG_LIB=paper_1204_5072_b200/_lib/variants/$n/liblfg.so timeout 900 \
      python -m pytest $TESTS -x -q -m gpu > $OUT/pytest_$n.txt 2>&1
done
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc --no-c3"
for i in 1 2 3; do
  for pq in "1.0 0.0" "0.95 0.05"; do
    set -- $pq; P=$1; Q=$2; shift 2
    timeout 300 $B --p $P --q $Q > $OUT/main_p${P}_$i.json 2> /dev/null
    for v in paper_1204_5072_b200/_lib/variants/*/liblfg.so; do
      n=$(basename $(dirname $v))
      LFG_LIB=$v timeout 300 $B --p $P --q $Q > $OUT/${n}_p${P}_$i.json 2> /dev/null
    done
  done
done
for f in $OUT/*.json; do
  echo $(basename $f) $(python -c "import json;d=json.load(open('$f'));print(round(d['value'],1))" 2>&1 | tail -1)
done > $OUT/summary.txt

#!/usr/bin/env bash
# Full ncu capture of one KPZ phase launch for a library variant.
# Usage: bash scripts/ncu_kpz.sh TAG [variant-dir-or-empty] [L]
TAG=${1:-prof}; VAR=${2:-}; L=${3:-65536}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$VAR" ]; then export LFG_LIB=$PWD/paper_1204_5072_b200/_lib/variants/$VAR/liblfg.so; fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kpz_dtr_phase -s 6 -c 1 \
    -o $OUT/prof_kpz_${VAR:-main} -f python bench.py --L $L --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_${VAR:-main}.log 2>&1
echo "ncu exit $?" >> $OUT/ncu_${VAR:-main}.log

#!/usr/bin/env bash
# Ensemble probe of decomposition schemes (scripts/explore/dt_explore.cu) on one B200.
# Usage: bash scripts/explore/run_explore.sh TAG "name|args" ...
set -u
TAG=$1; shift
OUT=gpurun_out/explore/$TAG; mkdir -p $OUT
B=scripts/explore/dt_explore
[ -x $B ] || nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o $B scripts/explore/dt_explore.cu
for spec in "$@"; do
  name=${spec%%|*}; args=${spec#*|}
  timeout 900 $B $args --out $OUT/$name.json >> $OUT/log.txt 2>&1 || echo "$name failed" >> $OUT/log.txt
done
echo done > $OUT/DONE

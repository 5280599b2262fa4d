#!/usr/bin/env bash
# KMC statistical tier (GPU DT vs reference sequential) in both active modes.
TAG=${1:-kmc_stats}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for both in 0 1; do
  timeout 1500 python scripts/kmc_stat_validate.py --L 64 --t 200 --seeds 256 --ref-seeds 128 --both $both \
      --out $OUT/kmc_L64_both$both.json > $OUT/kmc_L64_both$both.txt 2>&1
done
echo done > $OUT/DONE

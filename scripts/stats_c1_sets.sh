#!/usr/bin/env bash
# C1 (L = 1024, p = 1, 1000 MCS) with more independent 64 + 64 seed sets, default plan:
# the null distribution of max|z| (reference vs reference) against GPU vs reference.
OUT=gpurun_out/stats_c1sets; mkdir -p $OUT
for b in 13000 17000 21000 25000 29000 33000; do
  timeout 900 python scripts/stat_validate.py --L 1024 --t 1000 --seeds 64 --ref-seeds 64 --seed-base $b \
      --out $OUT/C1_64_b$b.json > $OUT/C1_64_b$b.log 2>&1
done
echo done > $OUT/DONE

#!/usr/bin/env bash
# C2 (BASELINE configs[1]): KPZ DTr, L = 2^16, p = 1, q = 0, flat start, 10^4 MCS, 16 seeds on one
# B200 (GPU only: the reference would need ~69 days per seed).  W^2(t) at t = round(1.1^k).
TAG=${1:-stats_c2}; OUT=gpurun_out/$TAG; mkdir -p $OUT
T=${2:-10000}
timeout 2400 python scripts/stat_validate.py --L 65536 --t $T --seeds 16 --no-ref --save-samples --beta-lo 100 \
    --out $OUT/stats_C2.json > $OUT/stats_C2.txt 2>&1
echo "exit $?" >> $OUT/stats_C2.txt

#!/usr/bin/env bash
# Statistical tier runs (GPU DTr ensembles vs reference sequential ensembles on host cores).
TAG=${1:-stats}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -m paper_1204_5072_b200.build > $OUT/build.txt 2>&1
timeout 900 python scripts/stat_validate.py --L 256 --t 100 --seeds 1000 --out $OUT/stats_L256_p1.json > $OUT/stats_L256_p1.txt 2>&1
timeout 900 python scripts/stat_validate.py --L 512 --t 100 --seeds 400 --p 0.95 --q 0.05 --out $OUT/stats_L512_p095.json > $OUT/stats_L512_p095.txt 2>&1
timeout 1500 python scripts/stat_validate.py --L 1024 --t 1000 --seeds 64 --beta-lo 32 --out $OUT/stats_C1.json > $OUT/stats_C1.txt 2>&1
echo done > $OUT/DONE

#!/usr/bin/env bash
# Statistical tier for plan sub = 8: GPU ensembles against the reference ensembles
# already recorded (same seeds) by scripts/stats_r02.sh / round 1.
OUT=gpurun_out/stats_sub8; mkdir -p $OUT
S="python scripts/stat_validate.py --sub 8"
R=profiles/stats
timeout 1200 $S --L 1024 --t 1000 --seeds 64 --ref-json $R/r02/C1_64.json --out $OUT/C1_64.json > $OUT/C1_64.log 2>&1
timeout 1200 $S --L 1024 --t 1000 --seeds 64 --seed-base 5000 --ref-json $R/r02/C1_64_b5000.json --out $OUT/C1_64_b5000.json > $OUT/C1_64_b5000.log 2>&1
timeout 1200 $S --L 1024 --t 1000 --seeds 64 --seed-base 9000 --ref-json $R/r02/C1_64_b9000.json --out $OUT/C1_64_b9000.json > $OUT/C1_64_b9000.log 2>&1
timeout 1200 $S --L 1024 --t 1000 --seeds 128 --ref-json $R/r02/C1_128.json --out $OUT/C1_128.json > $OUT/C1_128.log 2>&1
timeout 900 $S --L 256 --t 100 --seeds 4000 --ref-json $R/stats_L256_p1_4000.json --out $OUT/L256_4000.json > $OUT/L256_4000.log 2>&1
timeout 900 $S --L 2048 --t 100 --seeds 400 --ref-json $R/stats_L2048_p1_400_b1024x128.json --out $OUT/L2048_400.json > $OUT/L2048_400.log 2>&1
timeout 900 $S --L 512 --t 100 --p 0.95 --q 0.05 --seeds 400 --ref-json $R/r02/L512_p095.json --out $OUT/L512_p095.json > $OUT/L512_p095.log 2>&1
echo done > $OUT/DONE

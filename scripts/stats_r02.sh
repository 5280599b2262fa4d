#!/usr/bin/env bash
# Statistical tier, round 2 (default plan: sub = 4).  GPU DTr ensembles vs the
# unmodified reference's kpz_sweep_sequential (oracle/_ref) on the host cores.
OUT=gpurun_out/stats_r02; mkdir -p $OUT
S=scripts/stat_validate.py
# C1: L = 1024, p = 1, 1000 MCS, 64 + 64 seeds (fresh reference ensemble)
timeout 1200 python $S --L 1024 --t 1000 --seeds 64 --ref-seeds 64 --save-samples --out $OUT/C1_64.json > $OUT/C1_64.log 2>&1
# L = 256, p = 1, 100 MCS: 4000 GPU realizations vs the stored 4000-realization reference ensemble
timeout 900 python $S --L 256 --t 100 --seeds 4000 --ref-json profiles/stats/stats_L256_p1_4000.json --out $OUT/L256_4000.json > $OUT/L256_4000.log 2>&1
# L = 2048 (production 1024 x 128 plan), p = 1, 100 MCS: 400 vs the stored 400-realization reference
timeout 900 python $S --L 2048 --t 100 --seeds 400 --ref-json profiles/stats/stats_L2048_p1_400_b1024x128.json --out $OUT/L2048_400.json > $OUT/L2048_400.log 2>&1
# L = 512, p = 0.95, q = 0.05 (configs[2]'s parameters), 400 + 400 fresh
timeout 900 python $S --L 512 --t 100 --p 0.95 --q 0.05 --seeds 400 --ref-seeds 400 --out $OUT/L512_p095.json > $OUT/L512_p095.log 2>&1
# C1 again with 128 + 128 (stricter)
timeout 1200 python $S --L 1024 --t 1000 --seeds 128 --ref-seeds 128 --out $OUT/C1_128.json > $OUT/C1_128.log 2>&1
echo done > $OUT/DONE

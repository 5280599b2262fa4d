OUT=gpurun_out/xq2; mkdir -p $OUT
timeout 2400 python scripts/stat_validate.py --L 256 --t 100 --seeds 16000 --ref-seeds 16000 --out $OUT/L256_q128.json > $OUT/L256_q128.log 2>&1
for q in 32 1; do
  LFG_KPZ_XQ=$q timeout 900 python scripts/stat_validate.py --L 256 --t 100 --seeds 16000 --ref-json $OUT/L256_q128.json --out $OUT/L256_q$q.json > $OUT/L256_q$q.log 2>&1
done

OUT=gpurun_out/xq; mkdir -p $OUT
for q in 128 32 1; do
  LFG_KPZ_XQ=$q timeout 900 python scripts/stat_validate.py --L 256 --t 100 --seeds 4000 --ref-json profiles/stats/stats_L256_p1_4000.json --out $OUT/L256_q$q.json > $OUT/L256_q$q.log 2>&1
done

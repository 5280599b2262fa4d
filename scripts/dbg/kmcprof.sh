# KMC profiles (round 2, final kernels) + KMC sanitizer cases
OUT=gpurun_out/kprof; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmc_dt16p -s 20 -c 1 -o $OUT/pc256 -f python scripts/kmc_bench.py 256 3 > $OUT/ncu256.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmc_dt16_phase -s 20 -c 1 -o $OUT/q1024 -f python scripts/kmc_bench.py 1024 1 > $OUT/ncu1024.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kmc -c 60 --csv --log-file $OUT/launches256.csv python scripts/kmc_bench.py 256 3 > /dev/null 2>&1
S="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in racecheck memcheck synccheck initcheck; do
  for c in kmc_wide kmc_quad; do
    timeout 900 $S --tool $tool python scripts/sanitize_cases.py $c > $OUT/san_${tool}_$c.txt 2>&1; echo "$tool $c exit $?" >> $OUT/san_summary.txt
  done
  LFG_KMC_PC=0 timeout 900 $S --tool $tool python scripts/sanitize_cases.py kmc_wide1 > $OUT/san_${tool}_kmc_wide1.txt 2>&1; echo "$tool kmc_wide1 exit $?" >> $OUT/san_summary.txt
done

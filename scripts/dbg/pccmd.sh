OUT=gpurun_out/pc6; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmc_dt16p -s 20 -c 1 -o $OUT/pc256 python scripts/kmc_bench.py 256 3 > $OUT/ncu.log 2>&1; echo "ncu exit $?" >> $OUT/ncu.log

#!/usr/bin/env bash
# Full ncu capture of one KMC DT phase launch (L=256, default plan).
TAG=${1:-kmcprof}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmc_dt -s 20 -c 1 \
    -o $OUT/prof_kmc -f python scripts/kmc_bench.py 256 3 > $OUT/ncu_kmc.log 2>&1
echo "ncu exit $?" >> $OUT/ncu_kmc.log

OUT=gpurun_out/w2v4; mkdir -p $OUT
python scripts/w2_time.py 65536 50 > $OUT/w2_time.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpz_width_rows -s 2 -c 1 -o $OUT/w2 python scripts/w2_time.py 65536 2 > $OUT/ncu.log 2>&1; echo "ncu exit $?" >> $OUT/ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kpz_width -c 30 --csv --log-file $OUT/launches.csv python scripts/w2_time.py 65536 3 > /dev/null 2>&1

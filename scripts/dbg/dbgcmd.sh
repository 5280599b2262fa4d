T=r02f; mkdir -p gpurun_out/$T
python scripts/w2_time.py > gpurun_out/$T/w2_time.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpz_width_rows -c 1 -o gpurun_out/$T/prof_w2 -f python scripts/w2_time.py 65536 2 > gpurun_out/$T/ncu_w2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/$T/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-kmc --no-c3 > gpurun_out/$T/launches.log 2>&1
timeout 900 python bench.py > gpurun_out/$T/bench.json 2> gpurun_out/$T/bench.err
bash scripts/stats_c2.sh $T/c2

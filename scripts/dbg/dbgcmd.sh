T=r02r; mkdir -p gpurun_out/$T
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/$T/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-kmc --no-c3 > gpurun_out/$T/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kpz_dtr_phase -s 20 -c 1 -o gpurun_out/$T/prof_kpz -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-kmc --no-c3 > gpurun_out/$T/ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kpz_dtr_phase -s 20 -c 1 -o gpurun_out/$T/prof_kpz_p095 -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-kmc --no-c3 --p 0.95 --q 0.05 > gpurun_out/$T/ncu_p095.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmc_dt16w -s 16 -c 1 -o gpurun_out/$T/prof_kmc256 -f python scripts/kmc_bench.py 256 3 > gpurun_out/$T/ncu_kmc256.log 2>&1

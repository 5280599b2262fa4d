mkdir -p gpurun_out/v12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kpz_dtr_sweep -s 2 -c 1 -o gpurun_out/v12/prof_sweep -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-kmc > gpurun_out/v12/ncu.log 2>&1

T=r02h; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/$T/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/$T/pytest_gpu.txt
python scripts/w2_time.py > gpurun_out/$T/w2_time.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kpz_width -c 6 --csv --log-file gpurun_out/$T/w2_launches.csv python scripts/w2_time.py 65536 2 > /dev/null 2>&1
for L in 512 1024; do timeout 600 python scripts/kmc_bench.py $L 20 >> gpurun_out/$T/kmc_bench.txt 2>&1; done

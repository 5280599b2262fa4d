T=r02e; mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_sharded_capi_gpu.py -q > gpurun_out/$T/pytest_sharded.txt 2>&1; echo "exit $?" >> gpurun_out/$T/pytest_sharded.txt
python scripts/w2_time.py > gpurun_out/$T/w2_time.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpz_width_rows -c 1 -o gpurun_out/$T/prof_w2 -f python scripts/w2_time.py 65536 2 > gpurun_out/$T/ncu_w2.log 2>&1
bash scripts/dist_one_gpu.sh $T/dist > /dev/null 2>&1
S=scripts/stat_validate.py
timeout 900 python $S --L 1024 --t 1000 --seeds 64 --ref-seeds 64 --seed-base 5000 --out gpurun_out/$T/C1_64_b5000.json > gpurun_out/$T/C1_b5000.log 2>&1
timeout 900 python $S --L 1024 --t 1000 --seeds 64 --ref-seeds 64 --seed-base 9000 --out gpurun_out/$T/C1_64_b9000.json > gpurun_out/$T/C1_b9000.log 2>&1

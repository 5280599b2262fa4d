T=sub4d; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests/ -q -m gpu --durations=10 > gpurun_out/$T/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/$T/pytest_gpu.txt
for v in tma bulk; do
  if [ $v = bulk ]; then export LFG_KPZ_NO_TENSOR_MAP=1; fi
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-kmc > gpurun_out/$T/bench_$v.json 2>> gpurun_out/$T/bench.err
done
unset LFG_KPZ_NO_TENSOR_MAP
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kpz_dtr_phase -s 20 -c 1 -o gpurun_out/$T/prof_kpz -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-kmc --no-c3 > gpurun_out/$T/ncu.log 2>&1

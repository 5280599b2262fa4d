T=r02p; mkdir -p gpurun_out/$T
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc --no-c3"
for i in 1 2; do
  timeout 300 $B > gpurun_out/$T/main_$i.json 2>/dev/null
  LFG_LIB=$PWD/paper_1204_5072_b200/_lib/variants/base/liblfg.so timeout 300 $B > gpurun_out/$T/base_$i.json 2>/dev/null
  timeout 300 $B --p 0.95 --q 0.05 > gpurun_out/$T/main_p95_$i.json 2>/dev/null
  LFG_LIB=$PWD/paper_1204_5072_b200/_lib/variants/base/liblfg.so timeout 300 $B --p 0.95 --q 0.05 > gpurun_out/$T/base_p95_$i.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_kpz_gpu.py tests/test_writelog_gpu.py tests/test_scale_gpu.py tests/test_shard_gpu.py -q > gpurun_out/$T/pytest.txt 2>&1; echo "exit $?" >> gpurun_out/$T/pytest.txt

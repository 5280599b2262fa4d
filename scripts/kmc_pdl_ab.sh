mkdir -p gpurun_out/kw11
timeout 600 python -m pytest tests/test_kmc_gpu.py tests/test_shard_gpu.py tests/test_snapshot_gpu.py -x -q -m gpu > gpurun_out/kw11/pytest.txt 2>&1
for L in 256 512; do
  timeout 200 python scripts/kmc_bench.py $L 30 > gpurun_out/kw11/pdl_$L.txt 2>&1
  LFG_KMC_PDL=0 timeout 200 python scripts/kmc_bench.py $L 30 > gpurun_out/kw11/nopdl_$L.txt 2>&1
done

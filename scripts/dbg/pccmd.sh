OUT=gpurun_out/pc4; mkdir -p $OUT
timeout 200 python scripts/kmc_bench.py 256 30 > $OUT/pc_256.txt 2>&1
timeout 900 python -m pytest tests/test_kmc_gpu.py tests/test_writelog_gpu.py -x -q > $OUT/pytest.txt 2>&1; echo "exit $?" >> $OUT/pytest.txt

OUT=gpurun_out/sub8; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_kpz_gpu.py tests/test_writelog_gpu.py tests/test_sharded_capi_gpu.py -x -q > $OUT/pytest.txt 2>&1; echo "exit $?" >> $OUT/pytest.txt
timeout 600 python scripts/kpz_sub_perf.py > $OUT/perf.txt 2>&1
bash scripts/stats_sub8.sh

OUT=gpurun_out/q1; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kmc_gpu.py tests/test_writelog_gpu.py -x -q > $OUT/pytest.txt 2>&1; echo "exit $?" >> $OUT/pytest.txt
for q in 1 0; do for L in 512 1024; do LFG_KMC_Q=$q timeout 300 python scripts/kmc_bench.py $L 20 2>&1 | head -2 > $OUT/q${q}_$L.txt; done; done

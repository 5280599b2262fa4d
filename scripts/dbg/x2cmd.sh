OUT=gpurun_out/x2; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kmc_gpu.py tests/test_writelog_gpu.py tests/test_scale_gpu.py -x -q -k "kmc or KMC" > $OUT/pytest.txt 2>&1; echo "exit $?" >> $OUT/pytest.txt
for c in kmc_x2 kmc_quad; do timeout 300 python scripts/sanitize_cases.py $c >> $OUT/cases.txt 2>&1; done
for i in 1 2; do for x in 8192 0; do for L in 512 1024; do LFG_KMC_X2=$x timeout 300 python scripts/kmc_bench.py $L 10 2>&1 | head -2 > $OUT/x${x}_${L}_$i.txt; done; done; done
timeout 600 python scripts/slab_compute_proxy.py 1 > $OUT/slab_both.json 2>&1

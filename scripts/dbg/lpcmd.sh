OUT=gpurun_out/zc1; mkdir -p $OUT
LFG_KMC_ZC=1 timeout 900 python -m pytest tests/test_kmc_gpu.py -x -q > $OUT/pytest.txt 2>&1; echo "exit $?" >> $OUT/pytest.txt
LFG_KMC_ZC=1 timeout 300 python scripts/sanitize_cases.py kmc_quad > $OUT/quad.txt 2>&1; echo "exit $?" >> $OUT/quad.txt
for i in 1 2; do for z in 0 1; do for L in 512 1024; do LFG_KMC_ZC=$z timeout 300 python scripts/kmc_bench.py $L 10 2>&1 | head -2 > $OUT/z${z}_${L}_$i.txt; done; done; done
LFG_KMC_ZC=1 timeout 900 ncu --set full --clock-control none -k regex:kmc_dt16z -s 20 -c 1 -o $OUT/z1024 -f python scripts/kmc_bench.py 1024 1 > $OUT/ncu.log 2>&1

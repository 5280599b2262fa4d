T=r02s; mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/$T/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/$T/pytest_gpu.txt
for sub in 1 4; do
  for L in 256 1024; do
    python - <<PY >> gpurun_out/$T/kmc_perf.txt 2>&1
import json, sys, torch
sys.path.insert(0, '.')
import paper_1204_5072_b200 as lfg
st = torch.cuda.Stream()
for both in (True,):
    k = lfg.KmcLattice($L, 1.5, both, 7, sub=$sub)
    k.set_stream(st.cuda_stream); k.make_random_alloy(0.5, 3); k.sweep_async(3); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); k.sweep_async(10); e1.record(st); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"L": $L, "sub": $sub, "att_per_ns": ($L**3//2)*10/(ms*1e6)}))
    k.close()
PY
  done
done
timeout 1500 python scripts/kmc_stat_validate.py --L 64 --t 100 --seeds 1024 --ref-seeds 512 --both 1 --sub 4 --out gpurun_out/$T/kmc_L64_both1_sub4.json > gpurun_out/$T/kmc_sub4.txt 2>&1
timeout 1500 python scripts/kmc_stat_validate.py --L 64 --t 100 --seeds 1024 --ref-seeds 512 --both 1 --sub 1 --out gpurun_out/$T/kmc_L64_both1_sub1.json > gpurun_out/$T/kmc_sub1.txt 2>&1

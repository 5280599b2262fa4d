T=r02l; mkdir -p gpurun_out/$T
python scripts/sharded_one_gpu.py > gpurun_out/$T/sharded_one_gpu.txt 2>&1
bash scripts/sanitize.sh $T/san > /dev/null 2>&1

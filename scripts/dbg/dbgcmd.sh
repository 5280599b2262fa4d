T=r02m; mkdir -p gpurun_out/$T
python scripts/shard_compute_proxy.py > gpurun_out/$T/proxy_p1.json 2>&1
python scripts/shard_compute_proxy.py 0.95 0.05 > gpurun_out/$T/proxy_p095.json 2>&1

mkdir -p gpurun_out/d1
LFG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --L 4096 --steps 3 --warmup 1 --no-kmc --no-cpu-baseline > gpurun_out/d1/dist2_4096.json 2> gpurun_out/d1/dist2_4096.err
LFG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 3 --warmup 3 --no-kmc --no-cpu-baseline --no-e2e > gpurun_out/d1/dist2_default.json 2> gpurun_out/d1/dist2_default.err
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-kmc"
LFG_KPZ_SWEEP_KERNEL=1 timeout 300 $B > gpurun_out/d1/sweep6.json 2>/dev/null
LFG_LIB=$PWD/paper_1204_5072_b200/_lib/variants/minb5/liblfg.so LFG_KPZ_SWEEP_KERNEL=1 timeout 300 $B > gpurun_out/d1/sweep5.json 2>/dev/null
timeout 300 $B > gpurun_out/d1/phase.json 2>/dev/null

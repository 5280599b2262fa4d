#!/usr/bin/env bash
# The N>1 bench path (strip-sharded C3 lattice, PeerComm fused write-back push, device step
# barriers) with N ranks sharing ONE GPU: gloo for the host-side plumbing (NCCL refuses two
# ranks on one device), CUDA IPC peer mappings for the data path.  Exercises the multi-GPU
# code end to end; the numbers are not scaling figures (the ranks share one GPU's SMs).
TAG=${1:-dist1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for N in 2 4; do
  LFG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps 5 --warmup 3 \
      --no-kmc --no-cpu-baseline > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
  echo "N=$N exit $?" >> $OUT/summary.txt
  LFG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $((29700 + N)) bench.py --impl reference --gpus $N --steps 2 --warmup 1 \
      > $OUT/ref_n$N.json 2> $OUT/ref_n$N.err
  echo "ref N=$N exit $?" >> $OUT/summary.txt
done

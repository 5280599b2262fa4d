#!/usr/bin/env bash
# One GPU round-trip: parity tests, smoke, bench, ncu launch list + full capture.
# Usage (from the repo root, under gpurun):  bash scripts/gpu_check.sh [tag] [stages]
#   stages: comma list of test,smoke,bench,launches,ncu (default: all)
set -u
TAG=${1:-r01}
STAGES=${2:-test,smoke,bench,dist,launches,ncu}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
has() { [[ ",$STAGES," == *",$1,"* ]]; }

nvidia-smi -L > "$OUT/gpu.txt" 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> "$OUT/gpu.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1
free -g >> "$OUT/lscpu.txt" 2>&1

python -m paper_1204_5072_b200.build > "$OUT/build.txt" 2>&1 || echo "build failed" >> "$OUT/build.txt"

if has test; then
  timeout 900 python -m pytest tests/ -x -q -m gpu > "$OUT/pytest_gpu.txt" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.txt"
fi
if has smoke; then
  timeout 300 python __graft_entry__.py > "$OUT/smoke.txt" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.txt"
fi
if has bench; then
  timeout 900 python bench.py --steps 20 --warmup 3 > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?" >> "$OUT/bench.err"
fi
if has dist; then
  LFG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --L 4096 --steps 3 --warmup 1 \
      --no-kmc --no-cpu-baseline > "$OUT/dist2_gloo.json" 2> "$OUT/dist2_gloo.err"
  echo "dist exit $?" >> "$OUT/dist2_gloo.err"
fi
if has launches; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
      --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
      > "$OUT/launches.log" 2>&1
  echo "launches exit $?" >> "$OUT/launches.log"
fi
if has ncu; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:kpz_dtr_phase -s 6 -c 1 \
      -o "$OUT/prof_kpz" -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
      > "$OUT/ncu.log" 2>&1
  echo "ncu exit $?" >> "$OUT/ncu.log"
fi
echo done > "$OUT/DONE"

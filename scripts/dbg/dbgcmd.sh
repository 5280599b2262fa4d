mkdir -p gpurun_out/dbg2
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/dbg2/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/dbg2/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/dbg2/smoke.txt 2>&1; echo "smoke exit $?" >> gpurun_out/dbg2/smoke.txt
timeout 900 python bench.py > gpurun_out/dbg2/bench.json 2> gpurun_out/dbg2/bench.err; echo "bench exit $?" >> gpurun_out/dbg2/bench.err

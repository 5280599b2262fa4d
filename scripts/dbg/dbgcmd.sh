T=r02n; mkdir -p gpurun_out/$T
timeout 1200 python -m pytest tests/test_sharded_capi_gpu.py tests/test_cpp_dropin.py tests/test_kpz_gpu.py -q > gpurun_out/$T/pytest.txt 2>&1; echo "exit $?" >> gpurun_out/$T/pytest.txt

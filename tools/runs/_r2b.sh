mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_parity.py -x -q > gpurun_out/r2b_pytest.log 2>&1
tail -30 gpurun_out/r2b_pytest.log

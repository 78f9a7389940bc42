mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_device_barrier.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r2z14_pytest.log 2>&1
tail -3 gpurun_out/r2z14_pytest.log

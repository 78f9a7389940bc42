mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_device_barrier.py tests/test_gpu_peer.py -x -q > gpurun_out/r2z_pytest.log 2>&1
tail -5 gpurun_out/r2z_pytest.log

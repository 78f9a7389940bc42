mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullseq.py tests/test_gpu_router_tc.py tests/test_gpu_device_barrier.py tests/test_gpu_peer.py tests/test_gpu_dropin.py -x -q > gpurun_out/r2k_pytest.log 2>&1
tail -30 gpurun_out/r2k_pytest.log

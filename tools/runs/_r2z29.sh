timeout 900 python -m pytest tests/test_gpu_dropin_router.py tests/test_gpu_peer.py -q > gpurun_out/r2z29.log 2>&1; tail -30 gpurun_out/r2z29.log

timeout 1500 python -m pytest tests/test_gpu_fullseq.py tests/test_gpu_peer.py tests/test_gpu_device_barrier.py tests/test_gpu_parity.py -q -x > gpurun_out/r2v.log 2>&1; tail -3 gpurun_out/r2v.log

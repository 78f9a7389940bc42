timeout 900 python -m pytest tests/test_gpu_device_barrier.py -q -x > gpurun_out/r2q.log 2>&1; tail -3 gpurun_out/r2q.log

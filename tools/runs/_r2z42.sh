timeout 900 python -m pytest tests/test_gpu_device_barrier.py -x -q > gpurun_out/r2z42.log 2>&1; tail -3 gpurun_out/r2z42.log

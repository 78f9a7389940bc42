timeout 900 python -m pytest tests/test_gpu_device_barrier.py -x -q > gpurun_out/r2z28_db.log 2>&1; tail -2 gpurun_out/r2z28_db.log

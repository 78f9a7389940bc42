timeout 1200 python -m pytest tests/test_gpu_random_layers.py -q -rf > gpurun_out/r2z45.log 2>&1; tail -30 gpurun_out/r2z45.log

timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2z47.log 2>&1; tail -3 gpurun_out/r2z47.log

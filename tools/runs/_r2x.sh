timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gating_variants" > gpurun_out/r2x.log 2>&1; tail -15 gpurun_out/r2x.log

mkdir -p gpurun_out
timeout 600 python tools/router_bench.py --config c2 > gpurun_out/r2c_router_c2.log 2>&1
timeout 600 python tools/router_bench.py --config c4 > gpurun_out/r2c_router_c4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_router_tc.py tests/test_gpu_device_barrier.py -x -q > gpurun_out/r2c_pytest.log 2>&1
tail -30 gpurun_out/r2c_pytest.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest_all.log 2>&1
tail -5 gpurun_out/r2c_pytest_all.log

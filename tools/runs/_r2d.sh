mkdir -p gpurun_out
timeout 600 python tools/router_bench.py --config c2 > gpurun_out/r2d_router_c2.log 2>&1
timeout 600 python tools/router_bench.py --config c4 > gpurun_out/r2d_router_c4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_router_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/r2d_pytest.log 2>&1
tail -5 gpurun_out/r2d_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2d_bench.log 2>&1
tail -c 3000 gpurun_out/r2d_bench.log

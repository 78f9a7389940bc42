mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router_tc.py -x -q > gpurun_out/r2e_pytest.log 2>&1
tail -15 gpurun_out/r2e_pytest.log
timeout 600 python tools/router_bench.py --config c2 > gpurun_out/r2e_router_c2.log 2>&1
timeout 600 python tools/router_bench.py --config c4 > gpurun_out/r2e_router_c4.log 2>&1
cat gpurun_out/r2e_router_c2.log gpurun_out/r2e_router_c4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router_tc_kernel|router_wgrad_tc|combine_router" -c 3 -o gpurun_out/r2e_router -f python tools/router_bench.py --config c2 --reps 1 > gpurun_out/r2e_ncu.log 2>&1
tail -3 gpurun_out/r2e_ncu.log

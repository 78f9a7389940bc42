mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_router_tc.py tests/test_gpu_device_barrier.py tests/test_gpu_peer.py tests/test_gpu_fullseq.py tests/test_gpu_dropin.py -q -x > gpurun_out/r2s_pytest.log 2>&1
tail -3 gpurun_out/r2s_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2s_bench1.log 2>&1
tail -1 gpurun_out/r2s_bench1.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('1gpu', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"
B200MOE_E2E_CHECK=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2s_bench1b.log 2>&1
tail -1 gpurun_out/r2s_bench1b.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('1gpu nocheck', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"

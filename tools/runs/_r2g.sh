mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router_tc.py -x -q > gpurun_out/r2g_pytest.log 2>&1
tail -3 gpurun_out/r2g_pytest.log
timeout 600 python tools/router_bench.py --config c2 > gpurun_out/r2g_router_c2.log 2>&1
cat gpurun_out/r2g_router_c2.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2g_bench.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/r2g_bench.log').read().strip().splitlines()[-1]);r=d['roofline']
print(d['value'], d['ms_per_step'], d['e2e'], r['other_kernels_ms'], d['clocks'])"

mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2r_bench1.log 2>&1
tail -1 gpurun_out/r2r_bench1.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('1gpu', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'launches', d['gpu_launches'], 'frac', round(d['roofline']['frac'],3), 'clk', d['clocks'], 'cpu', d['cpu_baseline'])"
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2r_bench2.log 2>&1
tail -1 gpurun_out/r2r_bench2.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('2gpu', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'a2a', round(d['a2a']['busbw_gbs']), 'clk', d['clocks']['sm_mhz'])"

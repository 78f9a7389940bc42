# last full validation of the final code: 1 GPU suite + smoke + default bench (driver-like)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/fl_pytest.log 2>&1; tail -2 gpurun_out/fl_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fl_bench.log 2>&1
tail -1 gpurun_out/fl_bench.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('c2', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), r['frac'], d['cpu_baseline']['value'], d['gpu_launches'], d['clocks'])"
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/fl_ref.log 2>&1; tail -1 gpurun_out/fl_ref.log | cut -c1-160

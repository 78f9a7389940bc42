mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2y_pytest.log 2>&1
tail -3 gpurun_out/r2y_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; tail -2 gpurun_out/r2y_smoke.log
timeout 900 python bench.py > gpurun_out/r2y_bench.log 2>&1
tail -1 gpurun_out/r2y_bench.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print(round(d['value']), round(d['ms_per_step'],2), 'e2e', d['e2e'] and round(d['e2e']['value']), r['frac'], r.get('frac_of_burst'), d['cpu_baseline'], d['clocks'])"

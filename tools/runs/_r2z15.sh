mkdir -p gpurun_out
for cfg in c4 c5 c3; do
timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/r2z15_$cfg.log 2>&1
tail -1 gpurun_out/r2z15_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$cfg', round(d['value']), round(d['ms_per_step'],2), 'e2e', d['e2e'] and round(d['e2e']['value']), 'gemm', round(r['gemm_ms_per_step'],2), r['frac'], {k:v for k,v in r['other_kernels_ms'].items() if v>0.02}, d['clocks']['sm_mhz'])"
done

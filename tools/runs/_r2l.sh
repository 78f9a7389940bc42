mkdir -p gpurun_out
for cfg in c2 c3; do
  timeout 900 python bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/r2l_bench4_$cfg.log 2>&1
  tail -1 gpurun_out/r2l_bench4_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$cfg', d['n_gpus'], round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"
done

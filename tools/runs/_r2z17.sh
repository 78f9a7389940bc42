mkdir -p gpurun_out
for cfg in c4 c2; do
B200MOE_BENCH_DEBUG=1 timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/r2z18_$cfg.log 2>&1
grep allocator gpurun_out/r2z18_$cfg.log
tail -1 gpurun_out/r2z18_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$cfg', round(d['value']), round(d['ms_per_step'],2), 'e2e', d['e2e'] and round(d['e2e']['value']), 'gaps', r['launch_gaps_ms'], d['clocks']['sm_mhz'])"
done
GAPS=1 STEPS=4 PROBES=pipelined timeout 900 python tools/e2e_probe.py 2>&1 | grep -v Warn | head -30

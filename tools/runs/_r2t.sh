for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2t_bench1.log 2>&1
tail -1 gpurun_out/r2t_bench1.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('1gpu', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],2), 'gaps', round(d['roofline']['launch_gaps_ms'],3), 'clk', d['clocks']['sm_mhz'])"
done

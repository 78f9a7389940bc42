mkdir -p gpurun_out
summ() { tail -1 $1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];a=d['a2a'] or {};print('$2', d['n_gpus'], round(d['value']), round(d['ms_per_step'],2), 'e2e', d['e2e'] and round(d['e2e']['value']), 'push', round(a.get('ms_per_step',0),3), round(a.get('busbw_gbs',0)), 'bar', r['ep_barrier_ms'], 'clk', d['clocks']['sm_mhz'], 'frac', round(r['frac'],3))"; }
timeout 900 python bench.py --gpus 4 --config c5 --steps 10 --warmup 3 --no-cpu > gpurun_out/f4b_bench_c5.log 2>&1
summ gpurun_out/f4b_bench_c5.log c5
for cfg in c3 c4; do
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python bench.py --gpus 2 --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/f4b_bench2_$cfg.log 2>&1
summ gpurun_out/f4b_bench2_$cfg.log $cfg
done

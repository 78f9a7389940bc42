# round-2 final evidence, 4 x B200 (and 2 of them)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/f4_multi.log 2>&1; tail -2 gpurun_out/f4_multi.log
summ() { tail -1 $1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];a=d['a2a'] or {};print('$2', d['n_gpus'], round(d['value']), round(d['ms_per_step'],2), 'e2e', d['e2e'] and round(d['e2e']['value']), 'push', round(a.get('ms_per_step',0),3), round(a.get('busbw_gbs',0)), 'bar', r['ep_barrier_ms'], 'gaps', round(r['launch_gaps_ms'],3), 'clk', d['clocks']['sm_mhz'], 'frac', round(r['frac'],3))"; }
for cfg in c2 c3 c4; do
  timeout 900 python bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/f4_bench_$cfg.log 2>&1
  summ gpurun_out/f4_bench_$cfg.log "$cfg"
done
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/f4_bench2_c2.log 2>&1
summ gpurun_out/f4_bench2_c2.log "c2"
timeout 900 python bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/f4_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/f4_ref.log | cut -c1-200

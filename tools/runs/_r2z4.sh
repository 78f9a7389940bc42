mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r2z4_multi.log 2>&1
tail -3 gpurun_out/r2z4_multi.log
summ() { tail -1 $1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];a=d['a2a'] or {};print('$2', d['n_gpus'], round(d['value']), round(d['ms_per_step'],2), 'e2e', d['e2e'] and round(d['e2e']['value']), 'push', round(a.get('ms_per_step',0),3), round(a.get('busbw_gbs',0)), 'exp', a.get('expand_ms_per_step'), 'bar', r['ep_barrier_ms'], 'clk', d['clocks']['sm_mhz'], 'gemm', round(r['gemm_ms_per_step'],2))"; }
for cfg in c2 c4 c3; do
 for ov in 1 0; do
  B200MOE_PUSH_OVERLAP=$ov timeout 900 python bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2z4_${cfg}_ov$ov.log 2>&1
  summ gpurun_out/r2z4_${cfg}_ov$ov.log "$cfg ov=$ov"
 done
done

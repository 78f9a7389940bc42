summ() { tail -1 $1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];a=d['a2a'] or {};print('$2', round(d['value']), round(d['ms_per_step'],2), 'push', round(a.get('ms_per_step',0),3), 'bar', [round(v,2) for v in r['ep_barrier_ms']], 'gemm', round(r['gemm_ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"; }
for cfg in c3 c5 c2; do
for rep in 1 2; do
for v in "0 1" "1 8"; do
  set -- $v
  B200MOE_PUSH_OVERLAP=$1 B200MOE_PUSH_BLOCKS_PER_SM=$2 timeout 900 python bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2z37.log 2>&1
  summ gpurun_out/r2z37.log "$cfg ov=$1 bps=$2"
done
done
done

# N = 1, 2, 4 back to back on one 4-GPU box (driver-like SCALE series, C2)
summ() { tail -1 $1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];a=d['a2a'] or {};print('N=$2', round(d['value']), round(d['ms_per_step'],2), 'e2e', d['e2e'] and round(d['e2e']['value']), 'frac', round(r['frac'],3), 'push', a.get('busbw_gbs') and round(a['busbw_gbs']), 'clk', d['clocks']['sm_mhz'])"; }
for n in 1 2 4; do
  if [ $n = 1 ]; then timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > gpurun_out/fs_$n.log 2>&1
  else timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/fs_$n.log 2>&1; fi
  summ gpurun_out/fs_$n.log $n
done

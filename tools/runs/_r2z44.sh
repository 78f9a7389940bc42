timeout 1200 python tools/gemm_bench.py --routed --only "dgrad1 store" --reps 12 --burst 4 --variants "B200MOE_TAIL_SPLIT=0,B200MOE_TAIL_SPLIT=1" 2>&1 | grep -v Warn | tail -3
timeout 1200 python tools/gemm_bench.py --routed --only "fwd" --reps 12 --burst 4 --variants "B200MOE_TAIL_SPLIT=0,B200MOE_TAIL_SPLIT=1" 2>&1 | grep -v Warn | tail -5
for i in 1 2; do for v in 0 1; do
B200MOE_TAIL_SPLIT=$v timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2z44.log 2>&1
tail -1 gpurun_out/r2z44.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('c2 split=$v', round(d['value']), round(d['ms_per_step'],2), 'gemm', round(r['gemm_ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"
done; done

B200MOE_GEMM_ALIGN=64 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2z27_pytest64.log 2>&1; tail -2 gpurun_out/r2z27_pytest64.log
for i in 1 2; do
for al in 128 64; do
B200MOE_GEMM_ALIGN=$al timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2z27_$al.log 2>&1
tail -1 gpurun_out/r2z27_$al.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('align $al', round(d['value']), round(d['ms_per_step'],2), 'gemm', round(r['gemm_ms_per_step'],2), d['clocks']['sm_mhz'])"
done
done

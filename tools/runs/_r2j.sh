mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_pytest.log 2>&1
tail -3 gpurun_out/r2j_pytest.log
grep -h "dedup push" gpurun_out/r2j_pytest.log | head -3
for cfg in c2 c4 c3; do
  timeout 900 python bench.py --gpus 4 --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/r2j_bench4_$cfg.log 2>&1
  tail -1 gpurun_out/r2j_bench4_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$cfg', d['n_gpus'], round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), 'a2a', d['a2a'] and round(d['a2a']['busbw_gbs']), 'bar', r['ep_barrier_ms'], 'clk', d['clocks']['sm_mhz'])"
done
B200MOE_SHARED_SIDE=0 timeout 900 python bench.py --gpus 4 --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2j_bench4_c4_noside.log 2>&1
tail -1 gpurun_out/r2j_bench4_c4_noside.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('c4 noside', round(d['value']), round(d['ms_per_step'],2), r['ep_barrier_ms'], d['clocks']['sm_mhz'])"
timeout 600 python tools/nvlink_probe.py --gpus 4 > gpurun_out/r2j_nvprobe.log 2>&1
timeout 1200 ncu --metrics nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum --csv -k regex:"ep_dispatch|gemm_tc" --log-file gpurun_out/r2j_nvl_ncu.csv python tools/nvlink_probe.py --gpus 4 > gpurun_out/r2j_nvl_ncu.log 2>&1
tail -2 gpurun_out/r2j_nvl_ncu.log

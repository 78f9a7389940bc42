# round-2 final evidence, 1 x B200
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f1_pytest.log 2>&1
tail -3 gpurun_out/f1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1; tail -1 gpurun_out/f1_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/f1_bench_c2.log 2>&1
tail -1 gpurun_out/f1_bench_c2.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('c2', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), r['frac'], r['frac_of_burst'], d['cpu_baseline']['value'], d['clocks']['sm_mhz'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f1_ref.log 2>&1; tail -1 gpurun_out/f1_ref.log | cut -c1-300
for cfg in c3 c4 c5; do
timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/f1_bench_$cfg.log 2>&1
tail -1 gpurun_out/f1_bench_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$cfg', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), r['frac'], r['launch_gaps_ms'], d['clocks']['sm_mhz'])"
done
B200MOE_NCU_RANGE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/f1_launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/f1_ncu_launches.log 2>&1
tail -1 gpurun_out/f1_ncu_launches.log
B200MOE_NCU_RANGE=1 timeout 1800 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"gemm_tc|router_tc|combine|permute" -o gpurun_out/f1_step_full -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/f1_ncu_full.log 2>&1
tail -1 gpurun_out/f1_ncu_full.log
ls -la gpurun_out/ | head -40

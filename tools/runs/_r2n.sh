mkdir -p gpurun_out
for i in 1 2; do
for chk in 1 0; do
B200MOE_E2E_CHECK=$chk timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/r2n_e2e_$chk_$i.log 2>&1
tail -1 gpurun_out/r2n_e2e_$chk_$i.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('check=$chk', round(d['value']), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), 'clk', d['clocks']['sm_mhz'])"
done
done
B200MOE_PARITY_LOG=gpurun_out/r2n_fullsize.jsonl timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r2n_fullsize.log 2>&1
tail -3 gpurun_out/r2n_fullsize.log
for v in "B200MOE_PANEL_M=0" "B200MOE_PANEL_M=2" "B200MOE_PANEL_M=4" "B200MOE_PANEL_M=16"; do
  env $v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --csv -k regex:gemm_tc -c 2 python tools/gemm_bench.py --only dgrad1 --reps 1 --burst 1 > gpurun_out/r2n_pm_$v.csv 2>&1
  env $v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv -k regex:gemm_tc -c 2 python tools/gemm_bench.py --only fwd2 --reps 1 --burst 1 > gpurun_out/r2n_pmf_$v.csv 2>&1
done
timeout 900 python tools/gemm_bench.py --only dgrad1 --variants "B200MOE_PANEL_M=0,B200MOE_PANEL_M=2,B200MOE_PANEL_M=4,B200MOE_PANEL_M=16" --reps 5 > gpurun_out/r2n_pm_time.log 2>&1
timeout 900 python tools/gemm_bench.py --only fwd2 --variants "B200MOE_PANEL_M=0,B200MOE_PANEL_M=2,B200MOE_PANEL_M=4,B200MOE_PANEL_M=16" --reps 5 >> gpurun_out/r2n_pm_time.log 2>&1
cat gpurun_out/r2n_pm_time.log

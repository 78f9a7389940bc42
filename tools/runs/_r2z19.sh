mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q > gpurun_out/r2z19_pytest.log 2>&1; tail -2 gpurun_out/r2z19_pytest.log
timeout 900 python tools/gemm_bench.py --only "store" --reps 5 --burst 10 --variants "B200MOE_KSYNC=0,B200MOE_KSYNC=1;B200MOE_KSYNC_W=4;B200MOE_KSYNC_G=8,B200MOE_KSYNC=1;B200MOE_KSYNC_W=2;B200MOE_KSYNC_G=8,B200MOE_KSYNC=1;B200MOE_KSYNC_W=8;B200MOE_KSYNC_G=4" > gpurun_out/r2z19_bench.log 2>&1
cat gpurun_out/r2z19_bench.log
for v in 0 1; do
B200MOE_KSYNC=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -c 2 --csv --log-file gpurun_out/r2z19_ncu_$v.csv python tools/gemm_bench.py --only "dgrad1 store" --reps 1 --burst 1 > /dev/null 2>&1
grep -h "dram__bytes_read\|gpu__time" gpurun_out/r2z19_ncu_$v.csv | awk -F'","' '{print "ksync='$v'", $13, $15}'
done

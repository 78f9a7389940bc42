mkdir -p gpurun_out
for v in 0 1 2 4 8; do
  B200MOE_KSTAGGER=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv -k regex:gemm_tc -c 1 python tools/gemm_bench.py --only "dgrad1 store" --reps 1 --burst 1 > gpurun_out/r2o_ks_d_$v.csv 2>&1
  B200MOE_KSTAGGER=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv -k regex:gemm_tc -c 1 python tools/gemm_bench.py --only "fwd2" --reps 1 --burst 1 > gpurun_out/r2o_ks_f_$v.csv 2>&1
  grep -h "dram__bytes_read.sum\|lts__t_sector_hit" gpurun_out/r2o_ks_d_$v.csv gpurun_out/r2o_ks_f_$v.csv | awk -F'","' -v v=$v '{print "kstagger " v ": " $(NF-2) " " $NF}'
done
timeout 900 python tools/gemm_bench.py --variants "B200MOE_KSTAGGER=0,B200MOE_KSTAGGER=2,B200MOE_KSTAGGER=4,B200MOE_KSTAGGER=8" --reps 5 > gpurun_out/r2o_ks_time.log 2>&1
cat gpurun_out/r2o_ks_time.log

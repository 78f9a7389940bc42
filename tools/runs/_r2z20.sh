mkdir -p gpurun_out
for r in "" "--routed"; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -c 1 --csv --log-file gpurun_out/r2z20.csv python tools/gemm_bench.py --only "dgrad1 store" --reps 1 --burst 1 $r > gpurun_out/r2z20_$r.log 2>&1
grep -h "dram__bytes_read\|gpu__time\|cycles_elapsed" gpurun_out/r2z20.csv | awk -F'","' '{print "'$r'", $13, $15}'
grep routed gpurun_out/r2z20_$r.log
done

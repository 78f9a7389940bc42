timeout 900 ncu --set full --clock-control none -k regex:gemm_tc -c 1 -o gpurun_out/r2w_dgrad1 -f python tools/gemm_bench.py --only "dgrad1 store" --reps 1 --burst 1 > gpurun_out/r2w.log 2>&1
tail -2 gpurun_out/r2w.log
ncu --query-metrics 2>/dev/null | grep -i "fabric\|ltc" | head -40 > gpurun_out/r2w_fabric_metrics.txt

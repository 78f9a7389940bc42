mkdir -p gpurun_out
timeout 900 python tools/gemm_bench.py --reps 5 --burst 20 --variants "B200MOE_DEBUG_OPS=0,B200MOE_DEBUG_OPS=3" > gpurun_out/r2z11.log 2>&1
cat gpurun_out/r2z11.log

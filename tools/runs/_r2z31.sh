timeout 900 python tools/gemm_bench.py --routed --reps 3 --burst 10 --variants "B200MOE_CTA_GROUP=2,B200MOE_CTA_GROUP=1" 2>&1 | grep -v Warn | tail -10

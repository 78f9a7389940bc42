for kr in 7 0 7 0; do
B200MOE_ROUTER_KROT=$kr timeout 300 python tools/router_bench.py --config c2 --reps 30 2>&1 | grep router_fwd_fused | sed "s/^/krot=$kr /"
done
B200MOE_ROUTER_KROT=0 timeout 1200 python -m pytest tests/test_gpu_random_layers.py -q -k ep_split > gpurun_out/r2z46.log 2>&1; tail -3 gpurun_out/r2z46.log

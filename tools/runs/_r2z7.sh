mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_router_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/r2z8_pytest.log 2>&1
tail -2 gpurun_out/r2z8_pytest.log
for cfg in c2 c4; do
for ks in 1 2 4; do
for bm in 128 0; do
B200MOE_ROUTER_KSUB=$ks B200MOE_ROUTER_BM=$bm timeout 300 python tools/router_bench.py --config $cfg > gpurun_out/r2z8_${cfg}_${ks}_$bm.log 2>&1
echo "$cfg ks=$ks bm=$bm $(grep router_fwd_fused gpurun_out/r2z8_${cfg}_${ks}_$bm.log)"
done
done
done

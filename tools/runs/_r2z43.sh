timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_peer.py -x -q > gpurun_out/r2z43_pytest.log 2>&1; tail -2 gpurun_out/r2z43_pytest.log
timeout 900 python tools/gemm_bench.py --routed --reps 3 --burst 10 --variants "B200MOE_TAIL_SPLIT=0,B200MOE_TAIL_SPLIT=1" 2>&1 | grep -v Warn | tail -20

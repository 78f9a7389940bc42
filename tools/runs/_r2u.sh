STEPS=8 timeout 900 python tools/e2e_probe.py > gpurun_out/r2u_probe.log 2>&1
tail -20 gpurun_out/r2u_probe.log
STEPS=4 GAPS=1 timeout 900 python tools/e2e_probe.py > gpurun_out/r2u_gaps.log 2>&1
tail -30 gpurun_out/r2u_gaps.log

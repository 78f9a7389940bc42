mkdir -p gpurun_out
GAPS=1 STEPS=6 PROBES=direct,api timeout 900 python tools/e2e_probe.py > gpurun_out/r2z13_probe.log 2>&1
grep -v Warn gpurun_out/r2z13_probe.log | head -60

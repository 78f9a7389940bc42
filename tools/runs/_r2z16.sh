timeout 600 python tools/_syncprobe2.py c4 > gpurun_out/r2z16.log 2>&1; grep -v "^  File\|^    " gpurun_out/r2z16.log | head -30; grep -A24 "SYNC" gpurun_out/r2z16.log | head -80

mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_pytest.log 2>&1
tail -5 gpurun_out/r2i_pytest.log
grep -h "dedup push\|FAIL" gpurun_out/r2i_pytest.log | head
timeout 600 python tools/nvlink_probe.py --gpus 2 > gpurun_out/r2i_nvprobe.log 2>&1
tail -2 gpurun_out/r2i_nvprobe.log
timeout 900 ncu --metrics nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum --csv -k regex:"ep_dispatch|gemm_tc" --log-file gpurun_out/r2i_nvl_ncu.csv python tools/nvlink_probe.py --gpus 2 > gpurun_out/r2i_nvl_ncu.log 2>&1
tail -3 gpurun_out/r2i_nvl_ncu.log

mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r2h_topo.txt 2>&1
ncu --query-metrics 2>/dev/null | grep -i "nvl" > gpurun_out/r2h_nvl_metrics.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2h_pytest.log 2>&1
tail -5 gpurun_out/r2h_pytest.log
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2h_bench2.log 2>&1
tail -c 2500 gpurun_out/r2h_bench2.log
timeout 600 python tools/nvlink_probe.py --gpus 2 > gpurun_out/r2h_nvprobe.log 2>&1
cat gpurun_out/r2h_nvprobe.log | tail -2
M=$(awk '{print $1}' gpurun_out/r2h_nvl_metrics.txt | grep -E "^nvl(tx|rx)__bytes$|^nvlrx__bytes$|^nvltx__bytes$" | paste -sd, -)
echo "metrics: $M"
if [ -n "$M" ]; then
timeout 900 ncu --metrics $M.sum,gpu__time_duration.sum --csv -k regex:"ep_dispatch|gemm_tc" --log-file gpurun_out/r2h_nvl_ncu.csv python tools/nvlink_probe.py --gpus 2 > gpurun_out/r2h_nvl_ncu.log 2>&1
tail -3 gpurun_out/r2h_nvl_ncu.log
fi

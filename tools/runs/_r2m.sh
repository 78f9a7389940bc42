mkdir -p gpurun_out
B200MOE_NCU_RANGE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r2m_launches.csv python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/r2m_launch.log 2>&1
B200MOE_NCU_RANGE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"router_tc_kernel|router_wgrad_tc|combine_router|router_bwd|permute|combine" -o gpurun_out/r2m_router_full -f python bench.py --profile-only --steps 1 --warmup 3 > gpurun_out/r2m_full.log 2>&1
tail -2 gpurun_out/r2m_full.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2m_bench_c2.log 2>&1
tail -c 600 gpurun_out/r2m_bench_c2.log
for cfg in c4 c5; do timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu > gpurun_out/r2m_bench_$cfg.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2m_ref.log 2>&1
tail -c 400 gpurun_out/r2m_ref.log

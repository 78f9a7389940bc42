mkdir -p gpurun_out
for cv in 0 1; do
for b in 1 2; do
B200MOE_PUSH_CARVEOUT=$cv B200MOE_PUSH_BLOCKS_PER_SM=$b timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/push_overlap_probe.py > gpurun_out/r2z6_${cv}_$b.log 2>&1
grep "blocks/SM" gpurun_out/r2z6_${cv}_$b.log
done
done

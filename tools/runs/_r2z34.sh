for i in 1 2; do
timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/push_overlap_probe.py 2>&1 | grep "blocks/SM"
done

nvidia-smi topo -m 2>&1 | head -12
lscpu | grep -i "numa\|socket\|model name" 
for b in 0 1; do BIND=$b timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/numa_probe.py 2>&1 | grep -v Warn | grep "BIND\|rank\|aggregate"; done

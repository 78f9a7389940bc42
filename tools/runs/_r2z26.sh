for v in old new old new; do
  if [ $v = old ]; then cp paper_2504_14960_b200/libb200moe_old.so /tmp/lib.so; else cp paper_2504_14960_b200/libb200moe.so /tmp/lib.so; fi
  cp paper_2504_14960_b200/libb200moe.so /tmp/keep.so
  cp /tmp/lib.so paper_2504_14960_b200/libb200moe.so
  timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 tools/exchange_bench.py --topk 8 --experts 64 --hidden 3584 2>&1 | grep "push" | sed "s/^/$v /"
  cp /tmp/keep.so paper_2504_14960_b200/libb200moe.so
done

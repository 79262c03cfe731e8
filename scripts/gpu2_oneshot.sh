#!/bin/bash
# 2-GPU: one-shot vs two-shot data phase at P=2 over sizes (pipelined rounds).
OUT=gpurun_out/r2o
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
EC_ONESHOT_BYTES=4294967296 timeout 600 $TR --master-port 29931 -m paper_1908_04207_b200.harness sweep --flavors solo \
  --sizes 256K,1M,16M,100M,1G --out $OUT/oneshot.json > $OUT/oneshot.log 2>&1
EC_ONESHOT_BYTES=0 timeout 600 $TR --master-port 29932 -m paper_1908_04207_b200.harness sweep --flavors solo \
  --sizes 256K,1M,16M,100M,1G --out $OUT/twoshot.json > $OUT/twoshot.log 2>&1
EC_ONESHOT_BYTES=4294967296 timeout 600 $TR --master-port 29933 bench.py --gpus 2 --steps 50 --warmup 5 --no-extras > $OUT/bench_oneshot.log 2>&1
timeout 600 $TR --master-port 29934 bench.py --gpus 2 --steps 50 --warmup 5 --no-extras > $OUT/bench_twoshot.log 2>&1
echo done

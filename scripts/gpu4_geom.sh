#!/bin/bash
# 4-GPU: the allreduce sweep (solo + majority, 1 KiB - 1 GiB) and a TMA
# geometry sweep at 100 MB with two rounds in flight.  Outputs under gpurun_out/$TAG.
TAG=${TAG:-r2g}
OUT=gpurun_out/$TAG
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29712 -m paper_1908_04207_b200.harness sweep --flavors solo,majority \
  --sizes 1K,64K,1M,16M,100M,256M,1G --out $OUT/sweep4.json > $OUT/sweep4.log 2>&1
timeout 900 $TR --master-port 29713 -m paper_1908_04207_b200.harness sweep --flavors solo \
  --sizes 100M --workers 64,80,96,128 --chunks 8192,16384 --out $OUT/geom4.json > $OUT/geom4.log 2>&1
[ -n "$BENCH" ] && timeout 600 $TR --master-port 29715 bench.py --gpus 4 --steps 50 --warmup 5 > $OUT/bench4.log 2>&1
echo done

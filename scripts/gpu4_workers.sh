#!/bin/bash
# 4-GPU: worker-count choice for the step (bench, progressive update beside
# the round) and for plain rounds (100 MB sweep), two rounds in flight.
TAG=${TAG:-r2w}
OUT=gpurun_out/$TAG
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
for W in 80 96 128; do
  EC_WORKERS=$W timeout 300 $TR --master-port 2972$((W % 10)) bench.py --gpus 4 --steps 50 --warmup 5 --no-extras > $OUT/bench4_w$W.log 2>&1
done
timeout 900 $TR --master-port 29731 -m paper_1908_04207_b200.harness sweep --flavors solo,majority \
  --sizes 1K,64K,1M,100M --workers 96,112,128,144 --chunks 8192,16384 --out $OUT/geom4.json > $OUT/geom4.log 2>&1
echo done

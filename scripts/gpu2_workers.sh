#!/bin/bash
OUT=gpurun_out/r2w2
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29941 -m paper_1908_04207_b200.harness sweep --flavors solo \
  --sizes 16M,100M,1G --workers 96,128,144 --out $OUT/geom2.json > $OUT/geom2.log 2>&1
for W in 96 128; do
  EC_WORKERS=$W timeout 300 $TR --master-port 29942 bench.py --gpus 2 --steps 100 --warmup 5 --no-extras 2>&1 | grep '"metric"' | sed "s/^/EC_WORKERS=$W /" >> $OUT/steps.log
done
echo done

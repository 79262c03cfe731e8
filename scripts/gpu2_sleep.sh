#!/bin/bash
OUT=gpurun_out/r2sl
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
for NS in 512 64 512 64; do
  EC_IDLE_SLEEP_NS=$NS timeout 300 $TR --master-port 29996 bench.py --gpus 2 --steps 100 --warmup 5 --no-extras 2>&1 | grep '"metric"' | sed "s/^/EC_IDLE_SLEEP_NS=$NS /" >> $OUT/steps.log
done

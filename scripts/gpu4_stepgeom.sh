#!/bin/bash
# 4-GPU: TMA geometry for the eager-SGD step (progressive update beside the round).
OUT=gpurun_out/r2sg
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
run() { env "$@" timeout 300 $TR --master-port 29961 bench.py --gpus 4 --steps 100 --warmup 5 --no-extras 2>&1 | grep '"metric"' | sed "s/^/$* /" >> $OUT/steps.log; }
run EC_CHUNK=16384 EC_STAGES=2
run EC_CHUNK=8192 EC_STAGES=4
run EC_CHUNK=8192 EC_STAGES=3
run EC_CHUNK=8192 EC_STAGES=4 EC_WORKERS=96
run EC_CHUNK=16384 EC_STAGES=2
run EC_CHUNK=8192 EC_STAGES=4
echo done

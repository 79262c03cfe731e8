#!/bin/bash
# 4-GPU: arrival-word schedule for the progressive step update (bench --no-extras).
TAG=${TAG:-r2s}
OUT=gpurun_out/$TAG
mkdir -p $OUT
NP=${NP:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NP --master-addr 127.0.0.1"
for SIG in 0 -1 3 0 -1 3; do
  EC_SIGNAL_EVERY=$SIG timeout 300 $TR --master-port 29901 bench.py --gpus $NP --steps 100 --warmup 5 --no-extras >> $OUT/bench_sig$SIG.log 2>&1
done
echo done

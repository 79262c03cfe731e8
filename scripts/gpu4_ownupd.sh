#!/bin/bash
# 4-GPU (NP=2 or 4): the step with and without the owners' in-worker own-shard update.
NP=${NP:-4}
OUT=gpurun_out/r2ou$NP
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NP --master-addr 127.0.0.1"
run() { env "$@" timeout 300 $TR --master-port 29981 bench.py --gpus $NP --steps 100 --warmup 5 --no-extras 2>&1 | grep '"metric"' | sed "s/^/$* /" >> $OUT/steps.log; }
for i in 1 2; do
  run EC_OWN=on
  run EC_NO_OWN_UPDATE=1
done
echo done

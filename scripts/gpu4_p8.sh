#!/bin/bash
# 4-GPU box: P=8 as two ranks per GPU (functional: the P=8 geometry, 8 KiB
# chunks x 2 stages, the config-2/3 P=8 schedules at ResNet-50 size), then the
# N=4 bench line.  Outputs under gpurun_out/$TAG.
TAG=${TAG:-r2p8}
OUT=gpurun_out/$TAG
mkdir -p $OUT
EC_RANKS_PER_GPU=2 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 \
  --master-addr 127.0.0.1 --master-port 29951 tests/mp_check.py > $OUT/mp_check_p8.log 2>&1
echo rc=$? >> $OUT/mp_check_p8.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 \
  --master-port 29952 bench.py --gpus 4 --steps 50 --warmup 5 > $OUT/bench4.log 2>&1
echo done

#!/bin/bash
# Functional run of bench.py at N=8 on a 4-GPU box (two ranks per GPU: the
# engines time-slice, so the numbers are not measurements) and its reference
# arm.  gpurun_out/p8bench/
OUT=gpurun_out/p8bench; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1"
EC_RANKS_PER_GPU=2 timeout 1500 $TR --master-port 29711 bench.py --gpus 8 --steps 3 --warmup 3 > $OUT/bench_n8.log 2>&1; echo rc=$? >> $OUT/bench_n8.log
EC_RANKS_PER_GPU=2 timeout 600 $TR --master-port 29712 bench.py --gpus 8 --steps 3 --warmup 3 --impl reference > $OUT/bench_ref_n8.log 2>&1; echo rc=$? >> $OUT/bench_ref_n8.log

#!/bin/bash
# The checked build (device assertions) on a 4-GPU box: the GPU suite and
# mp_check at P=4.  gpurun_out/checked4/
OUT=gpurun_out/checked4; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
EC_DEBUG_LIB=1 timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $OUT/pytest_gpu_checked_4gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu_checked_4gpu.log
EC_DEBUG_LIB=1 timeout 1200 $TR --master-port 29731 tests/mp_check.py > $OUT/mp_check4_checked.log 2>&1; echo rc=$? >> $OUT/mp_check4_checked.log

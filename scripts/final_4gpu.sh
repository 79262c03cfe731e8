#!/bin/bash
# Final 4-GPU pass: mp_check (P=4 and P=8 as two ranks per GPU), the sweep,
# the N=4 bench line and its reference arm.  Outputs under gpurun_out/final4.
OUT=gpurun_out/final4
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29611 bench.py --gpus 4 --steps 50 --warmup 5 > $OUT/bench_n4.log 2>&1
timeout 600 $TR --master-port 29612 bench.py --gpus 4 --steps 10 --warmup 3 --impl reference > $OUT/bench_ref_n4.log 2>&1
timeout 600 $TR --master-port 29613 -m paper_1908_04207_b200.harness sweep --flavors solo,majority \
  --sizes 1K,64K,1M,16M,100M,256M,1G --out $OUT/sweep4.json > $OUT/sweep4.log 2>&1
timeout 900 $TR --master-port 29614 tests/mp_check.py > $OUT/mp_check4.log 2>&1; echo rc=$? >> $OUT/mp_check4.log
EC_RANKS_PER_GPU=2 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 \
  --master-addr 127.0.0.1 --master-port 29615 tests/mp_check.py > $OUT/mp_check_p8.log 2>&1
echo rc=$? >> $OUT/mp_check_p8.log
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 > $OUT/pytest_gpu_4gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu_4gpu.log
echo done

#!/bin/bash
# Final 2-GPU pass: the N=2 bench line and its reference arm, the sweep,
# mp_check at P=2 and the GPU suite.  Outputs under gpurun_out/final2.
OUT=gpurun_out/final2
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29621 bench.py --gpus 2 --steps 50 --warmup 5 > $OUT/bench_n2.log 2>&1
timeout 600 $TR --master-port 29622 bench.py --gpus 2 --steps 10 --warmup 3 --impl reference > $OUT/bench_ref_n2.log 2>&1
timeout 600 $TR --master-port 29623 -m paper_1908_04207_b200.harness sweep --flavors solo,majority \
  --sizes 1K,64K,1M,16M,100M,256M,1G --out $OUT/sweep2.json > $OUT/sweep2.log 2>&1
timeout 900 $TR --master-port 29624 tests/mp_check.py > $OUT/mp_check2.log 2>&1; echo rc=$? >> $OUT/mp_check2.log
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 > $OUT/pytest_gpu_2gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu_2gpu.log
echo done

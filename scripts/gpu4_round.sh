#!/bin/bash
# One 4-GPU measurement pass (gpurun --gpus 4): multi-process parity, the
# allreduce sweep with and without two rounds in flight, the NCCL yardstick
# and the N=4 bench line.  Outputs under gpurun_out/$TAG.
TAG=${TAG:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
if [ -z "$SKIP_MP" ]; then
  timeout 900 $TR --master-port 29611 tests/mp_check.py > $OUT/mp_check4.log 2>&1; echo rc=$? >> $OUT/mp_check4.log
fi
timeout 600 $TR --master-port 29612 -m paper_1908_04207_b200.harness sweep --flavors solo,majority \
  --sizes ${SIZES:-1K,64K,1M,16M,100M,256M,1G} --out $OUT/sweep4_lead2.json > $OUT/sweep4_lead2.log 2>&1
EC_NO_LEAD=1 timeout 600 $TR --master-port 29613 -m paper_1908_04207_b200.harness sweep --flavors solo,majority \
  --sizes 1K,1M,100M --out $OUT/sweep4_lead1.json > $OUT/sweep4_lead1.log 2>&1
[ -z "$SKIP_NCCL" ] && timeout 300 $TR --master-port 29614 scripts/nccl_yardstick.py > $OUT/nccl4.log 2>&1
EC_ONESHOT_BYTES=1048576 timeout 600 $TR --master-port 29617 -m paper_1908_04207_b200.harness sweep --flavors solo \
  --sizes 64K,256K,1M --out $OUT/sweep4_oneshot1m.json > $OUT/sweep4_oneshot1m.log 2>&1
EC_ONESHOT_BYTES=0 timeout 600 $TR --master-port 29618 -m paper_1908_04207_b200.harness sweep --flavors solo \
  --sizes 1K,64K --out $OUT/sweep4_twoshot.json > $OUT/sweep4_twoshot.log 2>&1
timeout 600 $TR --master-port 29615 bench.py --gpus 4 --steps 50 --warmup 5 > $OUT/bench4.log 2>&1
timeout 300 $TR --master-port 29616 scripts/nvlink_bytes.py > $OUT/nvlink_bytes.log 2>&1
echo done

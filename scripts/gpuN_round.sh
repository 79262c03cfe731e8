#!/bin/bash
# One multi-GPU measurement pass on NP GPUs (gpurun --gpus NP): multi-process
# parity (mp_check), the allreduce sweep (solo + majority, 1 KiB - 1 GiB), the
# NCCL yardstick, the bench line and NVLink byte counters.  Outputs under
# gpurun_out/$TAG.
NP=${NP:-4}
TAG=${TAG:-r2n$NP}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi topo -m > $OUT/topo.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NP --master-addr 127.0.0.1"
[ -z "$SKIP_MP" ] && { timeout 900 $TR --master-port 29811 tests/mp_check.py > $OUT/mp_check.log 2>&1; echo rc=$? >> $OUT/mp_check.log; }
timeout 600 $TR --master-port 29812 -m paper_1908_04207_b200.harness sweep --flavors solo,majority \
  --sizes ${SIZES:-1K,64K,1M,16M,100M,256M,1G} --out $OUT/sweep.json > $OUT/sweep.log 2>&1
[ -z "$SKIP_NCCL" ] && timeout 300 $TR --master-port 29814 scripts/nccl_yardstick.py > $OUT/nccl.log 2>&1
timeout 300 $TR --master-port 29816 scripts/nvlink_bytes.py > $OUT/nvlink_bytes.log 2>&1
timeout 600 $TR --master-port 29815 bench.py --gpus $NP --steps 50 --warmup 5 > $OUT/bench.log 2>&1
[ -n "$REF" ] && timeout 600 $TR --master-port 29817 bench.py --gpus $NP --steps 10 --warmup 3 --impl reference > $OUT/bench_ref.log 2>&1
echo done

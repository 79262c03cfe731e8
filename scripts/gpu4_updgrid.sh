#!/bin/bash
# The progressive update's grid vs the round's data phase in the N=4 step
# (EC_UPD_GRID caps the update kernel's CTAs).  gpurun_out/updgrid/
OUT=gpurun_out/updgrid; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
for g in 296 20 40 80 148 296; do
  EC_UPD_GRID=$g timeout 600 $TR --master-port $((29700 + RANDOM % 90)) bench.py --gpus 4 --steps 100 --warmup 10 --no-extras > $OUT/b_$g.log 2>&1
  echo "grid=$g $(grep '^{' $OUT/b_$g.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); t=d["timeline_us"]; print(round(d["value"]), round(d["ms_per_step"]*1e3,1), round(t["data_phase"],1), round(t["done_to_offer"],1), t["done_to_offer_detail"])')" >> $OUT/summary.txt
done

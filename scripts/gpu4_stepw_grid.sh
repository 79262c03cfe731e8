#!/bin/bash
# The step's worker count (EC_WORKERS_STEP) x the progressive update's grid
# (EC_UPD_GRID) at N=4.  gpurun_out/stepw/
OUT=gpurun_out/stepw; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
for cfg in "80 296" "96 296" "112 296" "128 296" "112 200" "128 200" "96 200" "80 296"; do
  set -- $cfg
  EC_WORKERS_STEP=$1 EC_UPD_GRID=$2 timeout 600 $TR --master-port $((29700 + RANDOM % 90)) bench.py --gpus 4 --steps 100 --warmup 10 --no-extras > $OUT/b_$1_$2.log 2>&1
  echo "w=$1 grid=$2 $(grep '^{' $OUT/b_$1_$2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); t=d["timeline_us"]; print(round(d["value"]), round(d["ms_per_step"]*1e3,1), round(t["data_phase"],1), round(t["done_to_offer"],1), round(t["done_to_offer_detail"]["done_to_update_report"],1))')" >> $OUT/summary.txt
done

#!/bin/bash
# The step's worker count (EC_WORKERS_STEP) at N=2.  gpurun_out/stepw2/
OUT=gpurun_out/stepw2; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
for w in 128 80 96 112 128 96; do
  EC_WORKERS_STEP=$w timeout 600 $TR --master-port $((29700 + RANDOM % 90)) bench.py --gpus 2 --steps 100 --warmup 10 --no-extras > $OUT/b_$w.log 2>&1
  echo "w=$w $(grep '^{' $OUT/b_$w.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); t=d["timeline_us"]; print(round(d["value"]), round(d["ms_per_step"]*1e3,1), round(t["data_phase"],1), round(t["done_to_offer"],1), round(t["done_to_offer_detail"]["done_to_update_report"],1))')" >> $OUT/summary.txt
done

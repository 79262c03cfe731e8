OUT=gpurun_out/exp54; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -q -m gpu --timeout 300 -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for e in side same side same; do
  if [ $e = same ]; then export EC_PUBLISH_SAME_STREAM=1; else unset EC_PUBLISH_SAME_STREAM; fi
  timeout 600 $TR --master-port $((29900 + RANDOM % 90)) bench.py --gpus 2 --steps 100 --warmup 10 --no-extras > $OUT/b_$e.log 2>&1
  echo "$e $(grep '^{' $OUT/b_$e.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["timeline_us"]["done_to_offer"], d["timeline_us"]["done_to_offer_detail"])')" >> $OUT/summary.txt
done

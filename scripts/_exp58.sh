OUT=gpurun_out/exp58; mkdir -p $OUT
for rep in 1 2; do
for e in base pre spin both; do
  unset EC_STEP_PREFETCH EC_STEP_SPIN
  case $e in pre) export EC_STEP_PREFETCH=1;; spin) export EC_STEP_SPIN=1;; both) export EC_STEP_PREFETCH=1 EC_STEP_SPIN=1;; esac
  timeout 300 python bench.py --no-extras --steps 300 --warmup 20 > $OUT/b_$e.log 2>&1
  echo "$e $(grep '^{' $OUT/b_$e.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')" >> $OUT/summary.txt
done; done

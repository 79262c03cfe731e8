#!/bin/bash
# compute-sanitizer over the engine (emulated P=2) and the direct step; logs
# under gpurun_out/san.  One GPU.
OUT=gpurun_out/san
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
export EC_TIMEOUT_S=120
for tool in racecheck synccheck memcheck; do
  for prog in engine direct; do
    timeout 900 $CS --tool $tool --print-limit 50 python scripts/sanitize_check.py $prog \
      > $OUT/${tool}_${prog}.log 2>&1
    echo "rc=$?" >> $OUT/${tool}_${prog}.log
  done
done
echo done

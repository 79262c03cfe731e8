#!/bin/bash
# Final 1-GPU pass: suite, smoke, bench lines, ncu launch lists and a full
# capture of the N=1 hot kernel.  Outputs under gpurun_out/final1.
OUT=gpurun_out/final1
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -q -m gpu --timeout 300 > $OUT/pytest_gpu.log 2>&1; echo rc=$? >> $OUT/pytest_gpu.log
[ -n "$CHECKED" ] && { EC_DEBUG_LIB=1 timeout 900 python -m pytest tests -q -m gpu --timeout 300 > $OUT/pytest_gpu_checked.log 2>&1; echo rc=$? >> $OUT/pytest_gpu_checked.log; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo rc=$? >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_n1.log 2>&1; echo rc=$? >> $OUT/bench_n1.log
timeout 600 python bench.py --impl reference > $OUT/bench_ref_n1.log 2>&1; echo rc=$? >> $OUT/bench_ref_n1.log
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches_n1.csv python bench.py --no-extras --steps 10 --warmup 3 > $OUT/ncu_launches.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ec_direct_step -s 6 -c 1 \
  -o $OUT/prof_direct_step python bench.py --no-extras --steps 10 --warmup 3 > $OUT/ncu_full.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $OUT/ncu_smoke.log 2>&1
echo done

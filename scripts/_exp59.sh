OUT=gpurun_out/exp59; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_scale.py tests/test_gpu_spec.py -q -m gpu -k "direct or p1 or P1 or bench" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for rep in 1 2 3; do
  timeout 300 python bench.py --no-extras --steps 300 --warmup 20 > $OUT/b_$rep.log 2>&1
  echo "final $(grep '^{' $OUT/b_$rep.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')" >> $OUT/summary.txt
done
timeout 300 python bench.py > $OUT/bench_default.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:ec_direct_step -s 6 -c 1 -o $OUT/prof_direct_step python bench.py --no-extras --steps 10 --warmup 3 > $OUT/ncu_full.log 2>&1

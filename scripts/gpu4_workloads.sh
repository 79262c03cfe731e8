#!/bin/bash
# 4-GPU: the workload side -- config 1 (hyperplane eager-SGD, live, the three
# flavors) with its eagercoll-train-v1 CSV + JSONL, the latency / NAP bench
# with its eagercoll-bench-v1 CSV + JSONL, and config 4 (LSTM).
OUT=gpurun_out/r2wl
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29971 -m paper_1908_04207_b200.harness train --out $OUT/train_c1_p4 > $OUT/train_c1_p4.log 2>&1
timeout 900 $TR --master-port 29972 -m paper_1908_04207_b200.harness latency --delay linear_skew:1.0 --out $OUT/latency_p4 > $OUT/latency_p4.log 2>&1
timeout 900 $TR --master-port 29973 -m paper_1908_04207_b200.harness lstm > $OUT/lstm_c4_p4.log 2>&1
echo done

#!/bin/bash
# 2 GPUs: co-resident optimizer, span/pack serialised while co-resident
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29680
for cfg in "gpt1.3b --clip 0" "gpt1.3b --clip 0 --sm-budget 74" "llama7b --clip 1.0"; do
  port=$((port+1))
  timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg >> gpurun_out/r2h_overlap_n2.jsonl 2>> gpurun_out/r2h_overlap.err
done

#!/bin/bash
# 2 GPUs: co-resident optimizer + auto pre-barrier + co-resident post-norm update spans
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29650
for cfg in "gpt1.3b --clip 0 --adamw exact" "gpt1.3b --clip 0 --adamw fast" "llama7b --clip 1.0 --adamw exact" "llama7b --clip 1.0 --adamw fast"; do
  port=$((port+1))
  timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg >> gpurun_out/r2g_overlap_n2.jsonl 2>> gpurun_out/r2g_overlap.err
done

#!/bin/bash
# 2 GPUs: co-resident span threshold A/B (32 M default vs 256 M) in the training iteration
cd "$(dirname "$0")/.."
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29830
for rep in 1 2; do for cs in 33554432 268435456; do for cfg in "gpt1.3b --clip 0" "llama7b --clip 1.0"; do
  port=$((port+1))
  HOD_CORUN_SPAN=$cs timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg 2>> $O/r2q.err | grep "^{" | sed "s/^{/{\"corun_span\": $cs, /" >> $O/r2q_overlap_n2.jsonl
done; done; done

#!/bin/bash
# 2 GPUs: span threshold sweep for the TMA span kernel in step() (d=2, 1.3B and LLaMA-7B clip)
cd "$(dirname "$0")/.."
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29980
for cfg in "gpt1.3b" "llama7b"; do for sp in 134217728 268435456 536870912 1073741824; do for fs in 33554432 67108864; do
  port=$((port+1))
  HOD_FIRST_SPAN=$fs timeout 600 $TR --master-port $port bench.py --gpus 2 --config $cfg --span-numel $sp --steps 10 --warmup 3 --no-e2e --no-overlap --no-parity 2>> $O/r3c.err | grep '^{"metric"' | sed "s/^{/{\"span\": $sp, \"first\": $fs, /" >> $O/r3c_bench.jsonl
done; done; done

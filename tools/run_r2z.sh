#!/bin/bash
# 4 GPUs: the alternated overlap measurement at d=2/4 (overlap_bench + bench lines with the practical NVLink key)
cd "$(dirname "$0")/.."
O=gpurun_out
port=29960
for n in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  for cfg in "gpt1.3b --clip 0" "llama7b --clip 1.0"; do
    port=$((port+1))
    timeout 900 $TR --master-port $port tools/overlap_bench.py --config $cfg 2>> $O/r2z.err | grep "^{" >> $O/r2z_overlap.jsonl
  done
  port=$((port+1))
  timeout 900 $TR --master-port $port bench.py --gpus $n --steps 20 --warmup 5 --extras 0 2>> $O/r2z.err | grep '^{"metric"' >> $O/r2z_bench.jsonl
done

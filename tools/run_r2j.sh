#!/bin/bash
# 4 GPUs: co-resident overlap at d=4 (1.3B nvls, LLaMA-7B clip p2p, budget 0 vs auto) + the default N=4 bench line (extras)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29720
for cfg in "gpt1.3b --clip 0" "gpt1.3b --clip 0 --sm-budget 0" "llama7b --clip 1.0" "llama7b --clip 1.0 --sm-budget 0"; do
  port=$((port+1))
  timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg >> gpurun_out/r2j_overlap_n4.jsonl 2>> gpurun_out/r2j.err
done
port=$((port+1))
timeout 1200 $TR --master-port $port bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2j_bench_n4.json 2>> gpurun_out/r2j.err

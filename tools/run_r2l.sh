#!/bin/bash
# 4 GPUs: TMA vs register span kernel at d=4 (LLaMA-7B clip p2p, 1.3B p2p)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=29770
for t in 1 0; do for cfg in "--config llama7b" "--backend p2p"; do
  port=$((port+1))
  HOD_SPAN_TMA=$t timeout 600 $TR --master-port $port bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-overlap --extras 0 $cfg | sed "s/^{/{\"tma\": $t, /" >> gpurun_out/r2l_bench_n4.jsonl 2>> gpurun_out/r2l.err
done; done

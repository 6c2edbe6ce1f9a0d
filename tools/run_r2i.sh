#!/bin/bash
# 2 GPUs: evict-first streaming hints A/B (libhod.so vs libhod_nohint.so)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29700
for lib in libhod.so libhod_nohint.so; do
  export HOD_LIB=$PWD/paper_2312_03549_b200/$lib
  for k in adamw fused_d2; do
    timeout 300 python tools/corun_probe.py --kernel $k --grids 0,148 | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/r2i_corun.jsonl 2>> gpurun_out/r2i.err
  done
  for cfg in "gpt1.3b --clip 0" "llama7b --clip 1.0"; do
    port=$((port+1))
    timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/r2i_overlap_n2.jsonl 2>> gpurun_out/r2i.err
  done
  port=$((port+1))
  timeout 600 $TR --master-port $port bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-overlap --no-parity | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/r2i_bench_n2.jsonl 2>> gpurun_out/r2i.err
  timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-parity | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/r2i_bench_n1.jsonl 2>> gpurun_out/r2i.err
done

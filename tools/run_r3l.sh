#!/bin/bash
# 2 GPUs: TMA span kernel 1 CTA/SM x 2048-element tiles (default) vs 2 CTAs/SM x 1024 (libhod_t1k2.so)
cd "$(dirname "$0")/.."
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29780
for lib in libhod.so libhod_t1k2.so; do
  export HOD_LIB=$PWD/paper_2312_03549_b200/$lib
  for d in 2 4 8; do for mode in fused rs adamw_ag; do
    timeout 120 python tools/fused_emulated.py --d $d --mode $mode | sed "s/^{/{\"lib\": \"$lib\", /" >> $O/r3l_fused.jsonl 2>> $O/r3l.err
  done; done
  for rep in 1 2; do for cfg in gpt1.3b llama7b; do
    port=$((port+1))
    timeout 600 $TR --master-port $port bench.py --gpus 2 --config $cfg --steps 10 --warmup 3 --no-e2e --no-overlap --no-parity 2>> $O/r3l.err | grep '^{"metric"' | sed "s/^{/{\"lib\": \"$lib\", /" >> $O/r3l_bench.jsonl
  done; done
done

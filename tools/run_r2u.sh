#!/bin/bash
# 2 GPUs: overlap timelines (Chrome trace) for 1.3B and LLaMA-7B clip; N=2 overlap noise (3 bench reps)
cd "$(dirname "$0")/.."
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29901 tools/overlap_bench.py --config gpt1.3b --trace $O/r2u_trace_gpt1.3b_n2_r{rank}.json 2>> $O/r2u.err | grep "^{" >> $O/r2u_overlap.jsonl
timeout 600 $TR --master-port 29902 tools/overlap_bench.py --config llama7b --clip 1.0 --trace $O/r2u_trace_llama7b_clip_n2_r{rank}.json 2>> $O/r2u.err | grep "^{" >> $O/r2u_overlap.jsonl
for rep in 1 2 3; do
  timeout 600 $TR --master-port 2991$rep bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-parity 2>> $O/r2u.err | grep '^{"metric"' >> $O/r2u_bench_n2.jsonl
done

#!/bin/bash
# N GPUs: full-grid packs (default) vs co-resident packs (HOD_CORUN_PACK=1) in the overlapped iteration
cd "$(dirname "$0")/.."
O=gpurun_out
N=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29920
for rep in 1 2; do for cp in high normal; do for cfg in "gpt1.3b --clip 0" "llama7b --clip 1.0"; do
  port=$((port+1))
  HOD_OPT_PRIORITY=$cp timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg 2>> $O/r2w.err | grep "^{" | sed "s/^{/{\"prio\": \"$cp\", /" >> $O/r2w_overlap_n$N.jsonl
done; done; done

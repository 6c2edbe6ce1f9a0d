#!/bin/bash
# 4 GPUs: SM vs copy-engine vs mixed peer pulls at d=2 and d=4
cd "$(dirname "$0")/.."
O=gpurun_out
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2999$n \
    tools/mix_probe.py --mb 256 2>> $O/r3g.err | grep "^{" >> $O/r3g_mix.jsonl
done

#!/bin/bash
# 2 GPUs: measured vs simulated 1F1B timeline (StageEvent form); guard-zone harness self-test
cd "$(dirname "$0")/.."
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29991 tools/pipeline_vs_sim.py --scenario scenarios/gpt1p3b_pp2_dp1_node.json --micro 16 \
  --timeline $O/r3m_timeline_gpt1p3b_pp2.json 2>> $O/r3e.err | grep "^{" >> $O/r3m_pipe_sim.jsonl

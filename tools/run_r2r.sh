#!/bin/bash
# 2 GPUs: one-GPU emulated PP x DP / 1F1B tests; measured pipeline vs the reference simulator
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_emulated_pipeline_gpu.py tests/test_multigpu_gpu.py -m gpu -q -k "emulated or pipeline" > $O/r2r_tests.log 2>&1; echo "rc=$?" >> $O/r2r_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29851 tools/pipeline_vs_sim.py --scenario scenarios/gpt1p3b_pp2_dp1_node.json --micro 16 2>> $O/r2r.err | grep "^{" >> $O/r2r_pipe_sim_n2.jsonl

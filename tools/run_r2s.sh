#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29861 tools/pipeline_vs_sim.py --scenario scenarios/gpt1p3b_pp2_dp1_node.json --micro 16 2>> $O/r2s.err | grep "^{" >> $O/r2s_pipe_sim_n2.jsonl
timeout 600 python -m pytest tests/test_emulated_pipeline_gpu.py -m gpu -q > $O/r2s_tests.log 2>&1; echo "rc=$?" >> $O/r2s_tests.log

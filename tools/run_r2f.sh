#!/bin/bash
# 2 GPUs: co-resident optimizer during backward (sm_budget 0 / 148 / 74), 1.3B and LLaMA-7B clip
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29600
for cfg in "gpt1.3b --clip 0" "llama7b --clip 1.0"; do
  for b in 0 148 74; do
    port=$((port+1))
    timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg --sm-budget $b >> gpurun_out/r2f_overlap_n2.jsonl 2>> gpurun_out/r2f_overlap.err
  done
done
timeout 900 python -m pytest tests/test_emulated_optimizer_gpu.py tests/test_multigpu_gpu.py tests/test_module_integration_gpu.py -m gpu -q -x > gpurun_out/r2f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2f_tests.log

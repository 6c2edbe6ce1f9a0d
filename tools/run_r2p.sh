#!/bin/bash
# 2 GPUs: 100-step emulated tests, LLaMA block-stack timing (co-resident vs full GPU), ncu of every hot kernel
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_emulated_optimizer_gpu.py tests/test_emulated_ranks_gpu.py -m gpu -q -k "100_steps or d_way" > $O/r2p_tests.log 2>&1; echo "rc=$?" >> $O/r2p_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29810
for b in 148 0 148 0; do
  port=$((port+1))
  HOD_SM_BUDGET=$b timeout 900 $TR --master-port $port tests/module_worker.py --mode dist --check 0 --time-iters 5 --dim 2048 --layers 16 --heads 16 --ffn 5504 --vocab 32000 --tokens 8192 --seq 2048 --bucket 25000000 2>> $O/r2p.err | grep "^{" | sed "s/^{/{\"sm_budget\": $b, /" >> $O/r2p_module_n2.jsonl
done
bash tools/run_r2n.sh

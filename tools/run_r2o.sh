#!/bin/bash
# 2 GPUs: whole GPU suite (regression, TMA default + co-resident hooks) and the
# LLaMA block-stack iteration timing with the co-resident default vs full-GPU launches
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > $O/r2o_tests.log 2>&1; echo "rc=$?" >> $O/r2o_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for b in 148 0; do
  HOD_SM_BUDGET=$b timeout 900 $TR --master-port 2980$b tests/module_worker.py --mode dist --check 0 --time-iters 5 --dim 2048 --layers 16 --heads 16 --ffn 5504 --vocab 32000 --tokens 8192 --seq 2048 --bucket 25000000 | grep "^{" | sed "s/^{/{\"sm_budget\": $b, /" >> $O/r2o_module_n2.jsonl 2>> $O/r2o.err
done

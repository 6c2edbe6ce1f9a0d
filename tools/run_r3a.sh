#!/bin/bash
# 2 GPUs: co-resident span CTA width (128 default vs 256) x pack/span serialisation; emulated parity
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_emulated_optimizer_gpu.py tests/test_emulated_pipeline_gpu.py -m gpu -q -k "match_oracle or pipeline or scenario" > $O/r3a_tests.log 2>&1; echo "rc=$?" >> $O/r3a_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29970
for rep in 1 2; do for v in "128 1" "256 1" "128 0"; do set -- $v
  port=$((port+1))
  HOD_CORUN_THREADS=$1 HOD_CORUN_SERIAL=$2 timeout 900 $TR --master-port $port tools/overlap_bench.py --config gpt1.3b 2>> $O/r3a.err | grep "^{" | sed "s/^{/{\"threads\": $1, \"serial\": $2, /" >> $O/r3a_overlap_n2.jsonl
done; done

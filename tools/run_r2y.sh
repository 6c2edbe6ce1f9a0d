#!/bin/bash
# 2 GPUs: gentle co-resident pack (unroll 2, default) vs unroll 8 (HOD_PACK_GENTLE=0): probe, overlap; emulated parity
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_emulated_optimizer_gpu.py -m gpu -q -k "match_oracle" > $O/r2y_tests.log 2>&1; echo "rc=$?" >> $O/r2y_tests.log
for g in 1 0; do
  HOD_PACK_GENTLE=$g timeout 300 python tools/corun_probe.py --kernel pack --grids 148 | sed "s/^{/{\"gentle\": $g, /" >> $O/r2y_corun.jsonl 2>> $O/r2y.err
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29940
for rep in 1 2; do for g in 1 0; do for cfg in "gpt1.3b --clip 0" "llama7b --clip 1.0"; do
  port=$((port+1))
  HOD_PACK_GENTLE=$g timeout 600 $TR --master-port $port tools/overlap_bench.py --config $cfg 2>> $O/r2y.err | grep "^{" | sed "s/^{/{\"gentle\": $g, /" >> $O/r2y_overlap_n2.jsonl
done; done; done

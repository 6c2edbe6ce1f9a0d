#!/bin/bash
# 2 GPUs: TMA span kernel — emulated parity tests, per-kernel A/B (one GPU, peers emulated), step A/B at N=2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_emulated_ranks_gpu.py tests/test_emulated_optimizer_gpu.py -m gpu -q -x -k "d_way or tma" > gpurun_out/r2k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k_tests.log
for d in 2 4 8; do for mode in fused rs adamw_ag; do for t in 0 1; do
  HOD_SPAN_TMA=$t timeout 120 python tools/fused_emulated.py --d $d --mode $mode | sed "s/^{/{\"tma\": $t, /" >> gpurun_out/r2k_fused.jsonl 2>> gpurun_out/r2k.err
done; done; done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29750
for t in 1 0; do for cfg in "" "--config llama7b"; do
  port=$((port+1))
  HOD_SPAN_TMA=$t timeout 600 $TR --master-port $port bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-overlap $cfg | sed "s/^{/{\"tma\": $t, /" >> gpurun_out/r2k_bench_n2.jsonl 2>> gpurun_out/r2k.err
done; done

#!/bin/bash
# round-2, 2 GPUs: new tests, TMA peer-read probe, exact vs fast AdamW in the step and the overlap
cd "$(dirname "$0")/.."
python -m pytest tests/test_module_integration_gpu.py tests/test_kernels_gpu.py tests/test_emulated_optimizer_gpu.py tests/test_optimizer_gpu.py -m gpu -q -k "fast or llama or long_pack" --timeout 900 > gpurun_out/r2b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_tests.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$TR --master-port 29521 tools/peer_bw.py --ops read,both,tma_read,tma_both --mb 256 > gpurun_out/r2b_peer_bw_n2.jsonl 2> gpurun_out/r2b_peer_bw.err
for mode in exact fast; do
  $TR --master-port 2953${#mode} bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --adamw $mode > gpurun_out/r2b_bench_n2_$mode.log 2>&1
done
for mode in exact fast; do
  $TR --master-port 2954${#mode} tools/overlap_bench.py --config gpt1.3b --adamw $mode > gpurun_out/r2b_ovl_n2_$mode.log 2>&1
done
$TR --master-port 29551 tests/module_worker.py --mode dist --check 0 --time-iters 5 --dim 2048 --layers 16 --heads 16 --ffn 5504 --vocab 32000 --tokens 8192 --seq 2048 --bucket 25000000 > gpurun_out/r2b_module_timing_n2.log 2>&1

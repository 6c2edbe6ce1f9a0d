#!/bin/bash
# 4 GPUs: TMA RS tile 8192 (default build) vs 2048 (libhod_rs2k.so): parity tests + LLaMA-7B clip bench at N=2/4
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_emulated_ranks_gpu.py tests/test_emulated_optimizer_gpu.py -m gpu -q -k "d_way or tma" > $O/r2t_tests.log 2>&1; echo "rc=$?" >> $O/r2t_tests.log
port=29880
for rep in 1 2; do for lib in libhod.so libhod_rs2k.so; do for n in 2 4; do
  port=$((port+1))
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  HOD_LIB=$PWD/paper_2312_03549_b200/$lib timeout 600 $TR --master-port $port bench.py --gpus $n --config llama7b --steps 10 --warmup 3 --no-e2e --no-overlap --no-parity 2>> $O/r2t.err | grep '^{"metric"' | sed "s/^{/{\"lib\": \"$lib\", /" >> $O/r2t_bench.jsonl
done; done; done

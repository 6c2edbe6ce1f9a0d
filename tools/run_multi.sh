#!/bin/bash
# Multi-GPU evidence run (one box, N GPUs): GPU tests, bench lines, overlap.
#   gpurun --gpus N -- 'bash tools/run_multi.sh N TAG'
N=${1:-4}; TAG=${2:-r01}
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
[ "${SKIP_TESTS:-0}" = 1 ] || timeout 1200 python -m pytest tests/test_multigpu_gpu.py -x -q > $O/${TAG}_mgpu_tests_n$N.log 2>&1; tail -1 $O/${TAG}_mgpu_tests_n$N.log
timeout 300 $TR --master-port 29621 bench.py --gpus $N --steps 10 --warmup 3 > $O/${TAG}_bench_gpt_n$N.log 2>&1
timeout 600 $TR --master-port 29622 bench.py --gpus $N --config llama7b --steps 10 --warmup 3 > $O/${TAG}_bench_llama_n$N.log 2>&1
for pb in 0 1; do
timeout 600 $TR --master-port 2963$pb tools/overlap_bench.py --config gpt1.3b --iters 5 --pre-barrier $pb > $O/${TAG}_ovl_gpt_pb${pb}_n$N.log 2>&1
timeout 900 $TR --master-port 2964$pb tools/overlap_bench.py --config llama7b --clip 1.0 --iters 5 --pre-barrier $pb > $O/${TAG}_ovl_llama_pb${pb}_n$N.log 2>&1
done
grep -h '"metric"\|"exposed' $O/${TAG}_*_n$N.log | cut -c1-200

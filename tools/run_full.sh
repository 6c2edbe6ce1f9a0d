#!/bin/bash
# Full validation on one box with N GPUs: GPU test suite, smoke, bench lines at 1..N.
#   gpurun --gpus N -- 'bash tools/run_full.sh N TAG'
N=${1:-4}; TAG=${2:-r01}
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/${TAG}_gpu_tests.log 2>&1; tail -1 $O/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.log 2>&1; tail -1 $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench_gpt_n1.log 2>&1
timeout 600 python bench.py --config llama7b > $O/${TAG}_bench_llama_n1.log 2>&1
for n in 2 4; do
  [ $n -le $N ] || continue
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $TR --master-port 2950$n bench.py --gpus $n > $O/${TAG}_bench_gpt_n$n.log 2>&1
  timeout 900 $TR --master-port 2960$n bench.py --gpus $n --config llama7b > $O/${TAG}_bench_llama_n$n.log 2>&1
done
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_reference_n1.log 2>&1
for n in 2 4; do
  [ $n -le $N ] || continue
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 600 $TR --master-port 2970$n tools/overlap_bench.py --config gpt1.3b --iters 5 2>/dev/null | grep exposed > $O/${TAG}_ovl_gpt_n$n.jsonl
  timeout 900 $TR --master-port 2980$n tools/overlap_bench.py --config llama7b --clip 1.0 --iters 5 2>/dev/null | grep exposed > $O/${TAG}_ovl_llama_n$n.jsonl
done
grep -h '"metric"' $O/${TAG}_bench_*.log | cut -c1-160

#!/bin/bash
# Full validation on one box with N GPUs: GPU test suite, smoke, bench lines at 1..N
# (N > 1 lines carry the iteration exposure; the default line at N >= 4 also the
# LLaMA-7B clip target, config 4 and the config-5 sweep), the PP x DP scenario,
# the reference arm, the measured-vs-simulated pipeline iteration.
#   gpurun --gpus N -- 'bash tools/run_full.sh N TAG'
N=${1:-4}; TAG=${2:-r02}
O=gpurun_out
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/${TAG}_gpu_tests.log 2>&1; tail -1 $O/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${TAG}_smoke.log 2>&1; tail -1 $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench_gpt_n1.log 2>&1
timeout 600 python bench.py --config llama7b > $O/${TAG}_bench_llama_n1.log 2>&1
for n in 2 4; do
  [ $n -le $N ] || continue
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1"
  timeout 900 $TR --master-port 2950$n bench.py --gpus $n > $O/${TAG}_bench_gpt_n$n.log 2>&1
  timeout 900 $TR --master-port 2960$n bench.py --gpus $n --config llama7b > $O/${TAG}_bench_llama_n$n.log 2>&1
done
if [ $N -ge 4 ]; then
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
  timeout 900 $TR --master-port 29704 bench.py --gpus 4 --steps 5 --scenario scenarios/gpt13b_pp2_dp2_hybrid.json \
    > $O/${TAG}_bench_gpt13b_pp2dp2_n4.log 2>&1
  timeout 900 $TR --master-port 29714 tools/pipeline_vs_sim.py --scenario scenarios/gpt13b_pp2_dp2_hybrid.json --micro 8 --timeline $O/${TAG}_pipeline_timeline_gpt13b_n4.json \
    > $O/${TAG}_pipeline_vs_sim_gpt13b_n4.log 2>&1
fi
timeout 600 python bench.py --impl reference > $O/${TAG}_bench_reference_n1.log 2>&1
grep -h '"metric"' $O/${TAG}_bench_*.log | cut -c1-160

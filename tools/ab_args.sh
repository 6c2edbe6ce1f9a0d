#!/bin/bash
# bench.py with several argument sets on N GPUs (same box, back to back, 2 reps).
#   bash tools/ab_args.sh N "common args" "args A" "args B" ...
N=$1; COMMON=$2; shift 2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29850
for rep in 1 2; do
  for setting in "$@"; do
    port=$((port+1))
    timeout 600 $TR --master-port $port bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $COMMON $setting 2>/dev/null \
      | grep '"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N $COMMON | $setting |', round(d['ms_per_step'],3), {k:(round(x['ms_total']/d['steps'],2)) for k,x in d['kernels'].items()})"
  done
done

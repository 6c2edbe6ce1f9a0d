#!/bin/bash
# one GPU: every hot kernel once under ncu --set full, summarised on the box
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:'(pack|pack_adamw|pack_sumsq|adamw_vec|adamw_scalar|sumsq|span_tma|p2p_step)_kernel' -f -o /tmp/r2n_each \
  python tools/ncu_each.py > $O/r2n_each_order.txt 2> $O/r2n_each.err
python tools/ncu_summary.py --round r02 --out-dir $O --each /tmp/r2n_each.ncu-rep --each-order $O/r2n_each_order.txt \
  --note "one launch per hot kernel at bucket size, peers emulated on one GPU (tools/ncu_each.py), cold cache; span_tma = TMA-fed span kernel (full-GPU default), span_reg = register-streaming span kernel (co-resident / NVLS), here both at full grid" > $O/r2n_sum_each.log 2>&1
for k in span_tma_kernel p2p_step_kernel; do
  ncu -i /tmp/r2n_each.ncu-rep -k regex:$k --page details --csv > $O/r2n_details_$k.csv 2>/dev/null
done
ls -la $O/r2n_*

#!/bin/bash
# one GPU: round-2 ncu evidence — every hot kernel once (--set full), the N=1 launch list,
# and a --set full capture of the N=1 dominant kernel inside the bench.  Reports are
# summarised ON the box (gpurun copies back <= 64 MiB) and deleted.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:'_kernel' -f -o $O/r2m_each \
  python tools/ncu_each.py > $O/r2m_each_order.txt 2> $O/r2m_each.err
python tools/ncu_summary.py --round r02 --each $O/r2m_each.ncu-rep --each-order $O/r2m_each_order.txt \
  --note "one launch per hot kernel at bucket size, peers emulated on one GPU (tools/ncu_each.py), cold cache" > $O/r2m_sum_each.log 2>&1
rm -f $O/r2m_each.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file $O/r2m_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity \
  > $O/r2m_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pack_adamw_kernel -s 150 -c 2 -f -o $O/r2m_pack_adamw \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > $O/r2m_ncu_pa.log 2>&1
python tools/ncu_summary.py --round r02 --launches $O/r2m_launches_n1.csv --rep pack_adamw=$O/r2m_pack_adamw.ncu-rep \
  --note "N=1 bench launch list (--metrics gpu__time_duration.sum) + --set full of pack_adamw_kernel inside the bench" > $O/r2m_sum.log 2>&1
ncu -i $O/r2m_pack_adamw.ncu-rep --page source --csv > $O/r2m_pack_adamw_source.csv 2>/dev/null
ls -la $O/r2m_*; du -sh $O

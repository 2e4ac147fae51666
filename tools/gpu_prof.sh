#!/bin/bash
# ncu campaign (one GPU): bench line, eager launch lists of one cycle (c2, c4 V(1,1); c2 W(1,0) reference defaults),
# --set full of each hot kernel (exported to CSV on the box; tools/ncu_summary.py turns them into profiles/).
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -f"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
for c in c2 c4; do
  SPAIMG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_$c.csv python tools/prof_op.py $c 9 2 > gpurun_out/ncu_l_$c.log 2>&1; echo launches_$c=$?
done
CYCLE=W NU1=1 NU2=0 CN=4 SPAIMG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches_c2_w10.csv python tools/prof_op.py c2 9 2 > gpurun_out/ncu_l_c2w.log 2>&1; echo launches_c2w=$?
for spec in "c2 0 sweep2d" "c2 1 residual_restrict2d" "c2 2 prolong" "c2 6 sweep2d" "c4 0 sweep3d" "c4 1 sweep3d" "c4 2 prolong" "c4 6 sweep3d"; do
  set -- $spec
  timeout 600 $NCU -k regex:$3 -s 2 -c 1 -o gpurun_out/full_$1_op$2 python tools/prof_op.py $1 $2 4 > gpurun_out/ncu_full_$1_$2.log 2>&1
  echo full_$1_$2=$?
done
# the coarse engine (inside an eager cycle)
SPAIMG_NO_GRAPH=1 timeout 600 $NCU -k regex:k_tail -s 1 -c 1 -o gpurun_out/full_c2_tail python tools/prof_op.py c2 9 2 > gpurun_out/ncu_full_tail.log 2>&1; echo full_tail=$?
# keep the merge-back small: export the reports to CSV on the box, drop the .ncu-rep files
for r in gpurun_out/full_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  rm -f $r
done
du -sh gpurun_out

#!/bin/bash
# ncu campaign (one GPU): eager launch list of one bench solve + --set full captures of each hot kernel.
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on -f"
SPAIMG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_c2.csv python tools/prof_op.py c2 9 1 > gpurun_out/ncu_l2.log 2>&1; echo l2=$?
SPAIMG_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/launches_c4.csv python tools/prof_op.py c4 9 1 > gpurun_out/ncu_l4.log 2>&1; echo l4=$?
for spec in "c2 0 sweep2d" "c2 1 residual_restrict2d" "c2 2 prolong" "c2 3 norm" "c4 0 sweep3d" "c4 1 ." "c4 2 prolong" "c4 3 ."; do
  set -- $spec
  timeout 600 $NCU -k regex:$3 -s 2 -c 2 -o gpurun_out/full_$1_op$2 python tools/prof_op.py $1 $2 4 > gpurun_out/ncu_full_$1_$2.log 2>&1
  echo full_$1_$2=$?
done

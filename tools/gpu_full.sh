#!/bin/bash
# One GPU campaign: gpu tests, bench line, ncu launch list of the bench, ncu full capture of K1.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep2d -s 3 -c 1 -o gpurun_out/prof_sweep2d -f \
  python tools/prof_op.py c2 0 5 > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?

mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python tools/prof_op.py c4 0 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep3d_march -s 1 -c 1 -o gpurun_out/prof_sweep3d -f python tools/prof_op.py c4 0 3 > gpurun_out/ncu.log 2>&1
echo ncu_rc=$?

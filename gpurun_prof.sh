mkdir -p gpurun_out
python tools/prof_op.py c2 0 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep2d_march -s 1 -c 1 -o gpurun_out/prof_sweep2d python tools/prof_op.py c2 0 3 > gpurun_out/ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu.log

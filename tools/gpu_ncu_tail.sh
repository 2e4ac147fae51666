mkdir -p gpurun_out
timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --warp-sampling-interval 0 --clock-control none --import-source on -f -k regex:k_tail -s 3 -c 1 -o gpurun_out/tailsrc python tools/prof_op.py c1 9 5 > gpurun_out/tailsrc.log 2>&1; echo ncu=$?
ncu -i gpurun_out/tailsrc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/tailsrc.source.csv 2>/dev/null
ncu -i gpurun_out/tailsrc.ncu-rep --page raw --csv > gpurun_out/tailsrc.raw.csv 2>/dev/null
rm -f gpurun_out/tailsrc.ncu-rep

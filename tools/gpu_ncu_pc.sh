mkdir -p gpurun_out
SPAIMG_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on -f --kernel-name-base demangled -k "regex:\(int\)3, \(bool\)0, \(int\)3" -s 1 -c 1 -o gpurun_out/pcsrc python tools/prof_op.py c2 9 2 > gpurun_out/pcsrc.log 2>&1; echo ncu=$?
ncu -i gpurun_out/pcsrc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pcsrc.source.csv 2>/dev/null
ncu -i gpurun_out/pcsrc.ncu-rep --page source --csv --print-source cuda > gpurun_out/pcsrc.cuda.csv 2>/dev/null
rm -f gpurun_out/pcsrc.ncu-rep
ls -la gpurun_out/pcsrc*

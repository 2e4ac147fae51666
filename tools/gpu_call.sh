mkdir -p gpurun_out
CYCLE=W NU1=1 NU2=0 CN=4 SPAIMG_NO_GRAPH=1 SPAIMG_TAIL_PROF=1 python tools/prof_op.py c1 9 2 > gpurun_out/tailprof_c1w.txt 2>&1
CYCLE=W NU1=1 NU2=0 CN=4 SPAIMG_NO_GRAPH=1 SPAIMG_TAIL_PROF=1 python tools/prof_op.py c3 9 2 > gpurun_out/tailprof_c3w.txt 2>&1
python tools/tune_w.py c2 SPAIMG_TAIL_FAST=1 > gpurun_out/tune_w_c2.txt 2>&1
python tools/tune_w.py c4 SPAIMG_TAIL_FAST=1 > gpurun_out/tune_w_c4.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?

mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
NU=2 SMOOTHER=m5 python tools/tune.py c2 SPAIMG_SWEEP2=0,1 > gpurun_out/tune_c2m5_nu2.txt 2>&1
NU=2 SMOOTHER=jacobi2d python tools/tune.py c2 SPAIMG_SWEEP2=0,1 > gpurun_out/tune_c2j_nu2.txt 2>&1

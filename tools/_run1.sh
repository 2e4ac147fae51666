timeout 1500 python -m pytest tests -m gpu -x -q -k "large_configs or alternate or fp32_cycles or medium" > gpurun_out/pytest_gpu_part.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_part.log
timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1 | cut -c1-80
NU=2 timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1| cut -c1-80
SMOOTHER=jacobi2d timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1| cut -c1-80
SMOOTHER=jacobi2d NU=2 timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1| cut -c1-80
SMOOTHER=m5 NU=2 timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1| cut -c1-80
bash tools/gpu_ncu_src.sh pc2 "k_sweep2d_march<double, \(int\)3, \(bool\)0, \(int\)3, \(bool\)0>" 1 c2 9 2 2>&1 | head -30 | cut -c1-200

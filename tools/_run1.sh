timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=0,512,256,128 2>&1 | tail -6
NU=2 timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=0,512,128 2>&1 | tail -6
SMOOTHER=jacobi3d timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=0,128 2>&1 | tail -6
timeout 600 python tools/tune.py c3 SPAIMG_PC3_N=0,128 2>&1 | tail -6
SPAIMG_PC3_N=512 bash tools/gpu_ncu_src.sh pc3 "k_sweep3d_march<double, \(int\)4, \(bool\)0, \(int\)4>" 1 c4 9 2 2>&1 | head -18
SPAIMG_PC3_N=0 bash tools/gpu_ncu_src.sh k13 "k_sweep3d_march<double, \(int\)4, \(bool\)0, \(int\)0>" 0 c4 9 2 2>&1 | head -18

timeout 900 python -m pytest tests -m gpu -x -q -k "pc3 or large_configs" > gpurun_out/pytest_gpu_part.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_part.log
timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=256 2>&1 | tail -1
NU=2 timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=256 2>&1 | tail -1
SMOOTHER=jacobi3d timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=256 2>&1 | tail -1
bash tools/gpu_ncu_src.sh pc3 "k_sweep3d_march<double, \(int\)4, \(bool\)0, \(int\)4>" 1 c4 9 2 2>&1 | head -18

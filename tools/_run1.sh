timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "large_configs or fp32_cycles or alternate" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -3
SMOOTHER=jacobi2d timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -3
NU=2 timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -3
bash tools/gpu_ncu_src.sh pc2 "k_sweep2d_march<double, \(int\)3, \(bool\)0, \(int\)3, \(bool\)0>" 1 c2 9 2 2>&1 | head -50

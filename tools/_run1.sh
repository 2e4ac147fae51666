timeout 900 python -m pytest tests -m gpu -x -q -k "large_configs or alternate or fp32_cycles or medium" > gpurun_out/pytest_gpu_part.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu_part.log
python tools/optime.py c2
timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1 | cut -c1-80
NU=2 timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1| cut -c1-80
SMOOTHER=jacobi2d timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1| cut -c1-80
SMOOTHER=jacobi2d NU=2 timeout 600 python tools/tune.py c2 SPAIMG_NO_GRAPH=0 2>&1 | tail -1| cut -c1-80

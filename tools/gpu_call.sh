set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python tools/tune_w.py c2 32,64 > gpurun_out/tune_w_c2.txt 2>&1
python tools/tune_w.py c1 32,64 > gpurun_out/tune_w_c1.txt 2>&1
python tools/tune_w.py c3 8,16 > gpurun_out/tune_w_c3.txt 2>&1
python tools/tune_w.py c4 8,16 > gpurun_out/tune_w_c4.txt 2>&1

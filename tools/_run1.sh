timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in c1 c2 c3 c4; do timeout 300 python tools/tune.py $c SPAIMG_NO_GRAPH=0 2>&1 | tail -1 | cut -c1-70; done
for c in c1 c2 c3 c4; do timeout 300 python tools/tune_w.py $c 64 2>&1 | tail -1 | cut -c1-70; done

timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2

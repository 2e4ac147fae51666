timeout 1500 python -m pytest tests -m gpu -x -q -k "pc3 or large_configs or medium or fp32 or generic or operators or cycles or alternate" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=0,256 2>&1 | tail -2
NU=2 timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=256 2>&1 | tail -1
SMOOTHER=jacobi3d timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=256 2>&1 | tail -1
timeout 600 python tools/tune.py c3 SPAIMG_PC3_N=0,128 2>&1 | tail -2
bash tools/gpu_ncu_src.sh pc3 "k_sweep3d_march<double, \(int\)4, \(bool\)0, \(int\)4>" 1 c4 9 2 2>&1 | head -18
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print(d['ms_per_cycle'], d['roofline']['frac'], d['e2e']['value'])
print(json.dumps(d['extra']['config5'], indent=0))
PY

timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=0,256 2>&1 | tail -2
NU=2 timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=256 2>&1 | tail -1
SMOOTHER=jacobi3d timeout 600 python tools/tune.py c4 SPAIMG_PC3_N=256 2>&1 | tail -1
timeout 600 python tools/tune.py c3 SPAIMG_PC3_N=0 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print(d['ms_per_cycle'], d['roofline']['frac'], d['e2e']['value'])
for k,v in d['extra']['config5'].items():
    if k.startswith('3d'): print(k, {kk: round(vv['frac'],3) for kk,vv in v.items()})
PY

"""Time solver cycles under different SPAIMG_* environment settings (read at solver creation).

    python tools/tune.py c2 SPAIMG_TAIL_N=0,16,32,64,128 [more VAR=a,b ...]

Prints ms per V-cycle (device-timed, solve loop to tolerance, median of 5) per setting,
and checks the residual history is identical across settings.
"""
import itertools
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from paper_2206_05543_b200 import workloads  # noqa: E402

cfg_id = sys.argv[1]
specs = [a.split("=", 1) for a in sys.argv[2:]]
names = [s[0] for s in specs]
values = [s[1].split(",") for s in specs]
sm, nu = {"c1": ("m9", 1), "c2": ("m9", 1), "c3": ("m7", 1), "c4": ("m7", 1)}[cfg_id]
if os.environ.get("SMOOTHER"):
    sm = os.environ["SMOOTHER"]
if os.environ.get("NU"):
    nu = int(os.environ["NU"])
dim, N, _ = workloads.CONFIGS[cfg_id]
b = torch.as_tensor(workloads.rhs(cfg_id)).cuda()
cfg = sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=nu, nu2=nu, coarsest_N=2, tol=1e-10)
ref = None
for combo in itertools.product(*values):
    for k, v in zip(names, combo):
        os.environ[k] = v
    s = sp.Solver(cfg, dim, N)
    s.load(b)
    ts = []
    for _ in range(6):
        s.load(None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hist, k, conv = s.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / k)
    st = s.stats()
    same = "ref" if ref is None else ("same" if hist == ref else f"DIFF max rel {max(abs(a - r) / r for a, r in zip(hist, ref)):.2e}")
    if ref is None:
        ref = hist
    print(f"{cfg_id} {sm} V({nu},{nu}) {dict(zip(names, combo))}: {np.median(ts[1:]):.4f} ms/cycle, {k} cycles, "
          f"{st['kernels_per_cycle']} kernels/cycle, history {same}", flush=True)
    del s
    torch.cuda.empty_cache()

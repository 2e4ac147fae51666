"""W-cycle (reference MgConfig defaults: W(1,0), coarsest_N=4) per-cycle time vs SPAIMG_TAIL_N
(or another SPAIMG_* switch).
    python tools/tune_w.py c2 32,64,128
    python tools/tune_w.py c2 SPAIMG_CLUSTER_N=0,64,256"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from paper_2206_05543_b200 import workloads  # noqa: E402

cid = sys.argv[1]
dim, N, _ = workloads.CONFIGS[cid]
sm = "m9" if dim == 2 else "m7"
b = torch.as_tensor(workloads.rhs(cid)).cuda()
cfg = sp.MgConfig(smoother=sp.named(sm))  # reference defaults: cycle="W", nu1=1, nu2=0, coarsest_N=4
var, vals = sys.argv[2].split("=", 1) if "=" in sys.argv[2] else ("SPAIMG_TAIL_N", sys.argv[2])
ref = None
for t in vals.split(","):
    os.environ[var] = t
    s = sp.Solver(cfg, dim, N)
    s.load(b)
    ts = []
    for _ in range(4):
        s.load(None)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        h, k, c = s.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / k)
    same = "ref" if ref is None else ("same" if h == ref else "DIFF")
    ref = ref or h
    print(f"{cid} {sm} W(1,0) cN=4 {var}={t}: {np.median(ts[1:]):.3f} ms/cycle, {k} cycles, "
          f"{s.stats()['kernels_per_cycle']} kernels/cycle, {same}", flush=True)
    del s

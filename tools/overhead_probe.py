"""Per-cycle time of the device-side solve loop vs plain cycle-graph replays (c1, c2, c3):
    SPAIMG_SOLVE_TAIL=1 / SPAIMG_SOLVE_IF=1 python tools/overhead_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from paper_2206_05543_b200 import workloads  # noqa: E402

for cid, sm in (("c1", "m9"), ("c2", "m9"), ("c3", "m7")):
    dim, N, _ = workloads.CONFIGS[cid]
    b = torch.as_tensor(workloads.rhs(cid)).cuda()
    cfg = sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=1, nu2=1, coarsest_N=2)
    s = sp.Solver(cfg, dim, N)
    s.load(b)
    for mode in ("run", "cycles"):
        ts = []
        for _ in range(5):
            s.load(None)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            if mode == "run":
                h, k, c = s.run()
            else:
                s.cycles(10)
                k = 10
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / k)
        print(cid, mode, f"{np.median(ts) * 1e3:.1f} us/cycle", k, "cycles" if mode == "run" else "", flush=True)

"""Solver.stats() (levels, launches per cycle, B_cycle) of the V(1,1) solve graph for c1-c4."""
import sys

import torch
sys.path.insert(0, '/root/repo')
import paper_2206_05543_b200 as sp
from paper_2206_05543_b200 import workloads
for cid, sm in (("c1","m9"),("c2","m9"),("c3","m7"),("c4","m7")):
    dim, N, _ = workloads.CONFIGS[cid]
    s = sp.Solver(sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=1, nu2=1, coarsest_N=2), dim, N)
    s.load(torch.zeros((N-1,)*dim, dtype=torch.float64, device="cuda")); s.run()
    print(cid, s.stats())

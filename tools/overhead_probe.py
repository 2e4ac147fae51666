import sys, os, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2206_05543_b200 as sp
from paper_2206_05543_b200 import workloads
for cid in ['c1','c2']:
    dim, N, _ = workloads.CONFIGS[cid]
    b = torch.as_tensor(workloads.rhs(cid)).cuda()
    cfg = sp.MgConfig(smoother=sp.named('m9'), cycle='V', nu1=1, nu2=1, coarsest_N=2)
    s = sp.Solver(cfg, dim, N); s.load(b)
    for mode in ["run", "cycles"]:
        ts=[]
        for _ in range(5):
            s.load(None)
            e0,e1=torch.cuda.Event(True),torch.cuda.Event(True)
            e0.record()
            if mode=='run': h,k,c = s.run()
            else: s.cycles(10); k=10
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)/k)
        print(cid, mode, f"{np.median(ts)*1e3:.1f} us/cycle", s.stats()['kernels_per_cycle'])

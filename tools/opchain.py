"""Per-launch time of each hot kernel replayed back to back in a CUDA graph, per level size.
    python tools/opchain.py 2 m9 64 128 256 512 1024 2048 4096"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402

dim, sm = int(sys.argv[1]), sys.argv[2]
for N in map(int, sys.argv[3:]):
    rng = np.random.default_rng(0)
    shape = (N - 1,) * dim
    x = torch.as_tensor(rng.uniform(-1, 1, shape)).cuda()
    b = torch.as_tensor(rng.uniform(-1, 1, shape)).cuda()
    cfg = sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=1, nu2=1, coarsest_N=2)
    s = sp.Solver(cfg, dim, N)
    s.load(b, x)
    out = []
    for op in range(4):
        reps = 200
        s.op(op, reps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        s.op(op, reps)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / reps * 1e3)
    print(f"dim {dim} N {N}: sweep {out[0]:.2f} us, res+restrict {out[1]:.2f} us, prolong+corr {out[2]:.2f} us, "
          f"norm {out[3]:.2f} us", flush=True)

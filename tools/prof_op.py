"""Launch one hot-path kernel in isolation for ncu: python tools/prof_op.py <cfg> <op> [reps] [dtype]
cfg: c2 (2D 4096^2 m9), c4 (3D 512^3 m7), c5_2d (16384^2 m9), c5_3d (512^3 m7); op: 0 sweep,
1 residual+restrict, 2 prolong+correct, 3 norm, 4 norm+sweep (part A), 5 two sweeps in one march,
6 K3+K1 (prolongation + correction fused into the sweep), 9 = whole
cycles."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from paper_2206_05543_b200 import workloads  # noqa: E402

cfg_id, op = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dtype = sys.argv[4] if len(sys.argv) > 4 else "float64"
spec = {"c2": (2, 4096, "m9"), "c4": (3, 512, "m7"), "c5_2d": (2, 16384, "m9"), "c5_3d": (3, 512, "m7"),
        "c1": (2, 256, "m9"), "c3": (3, 128, "m7")}[cfg_id]
dim, N, sm = spec
rng = np.random.default_rng(2)
shape = (N - 1,) * dim
x = torch.as_tensor(rng.uniform(-1, 1, shape)).cuda()
b = torch.as_tensor(rng.uniform(-1, 1, shape)).cuda()
if dtype == "float32":
    x, b = x.float(), b.float()
# CYCLE=W NU1=1 NU2=0 CN=4 selects the reference MgConfig defaults instead of V(1,1), cN=2
env = os.environ.get
cfg = sp.MgConfig(smoother=sp.named(sm), cycle=env("CYCLE", "V"), nu1=int(env("NU1", 1)), nu2=int(env("NU2", 1)),
                  coarsest_N=int(env("CN", 2)))
s = sp.Solver(cfg, dim, N, dtype=dtype)
s.load(b, x)
if op == 9:
    s.cycles(reps)
else:
    s.op(op, reps)
torch.cuda.synchronize()
print("done", cfg_id, op, reps, dtype, s.stats())

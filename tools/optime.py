"""Per-launch time of the hot operators replayed in a graph (Solver.op): python tools/optime.py c2|c4 [dtype]
ops: 0 sweep, 1 residual+restrict, 2 prolong+correct, 3 norm, 4 norm+sweep, 6 K3+K1."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from bench import time_events  # noqa: E402

cfg_id = sys.argv[1]
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
dim, N, sm = {"c2": (2, 4096, "m9"), "c4": (3, 512, "m7"), "c2j": (2, 4096, "jacobi2d"), "c4j": (3, 512, "jacobi3d")}[cfg_id]
rng = np.random.default_rng(2)
x = torch.as_tensor(rng.uniform(-1, 1, (N - 1,) * dim)).cuda()
b = torch.as_tensor(rng.uniform(-1, 1, (N - 1,) * dim)).cuda()
if dtype == "float32":
    x, b = x.float(), b.float()
so = sp.Solver(sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=1, nu2=1, coarsest_N=2), dim, N, dtype=dtype)
so.load(b, x)
stream = torch.cuda.current_stream()
esz = 8 if dtype == "float64" else 4
n = (N - 1) ** dim
for op, name, bpu in ((0, "sweep", 3.0), (1, "residual+restrict", 2 + 2.0 ** -dim), (2, "prolong+correct", 2 + 2.0 ** -dim),
                      (3, "norm", 2.0), (4, "norm+sweep", 3.0), (6, "K3+K1", 3 + 2.0 ** -dim)):
    so.op(op, 20)
    t = min(time_events(lambda: so.op(op, 20), stream, 20) for _ in range(5))
    print(f"{cfg_id} {dtype} op {op} {name:18s} {t * 1e6:8.2f} us  {bpu * esz * n / t / 1e12:.2f} TB/s")

"""Helper for test_gpu_parity.test_alternate_paths_bitwise (run in a subprocess so that the
library reads the SPAIMG_* switches fresh): zero-start V(1,1) solves of configs 1 and 3 and a
W(1,0) solve at N=64, printed as JSON {case: [iterations, norms, sha256(u)]}."""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from paper_2206_05543_b200 import workloads  # noqa: E402

out = {}
for case, (cfg_id, sm, cyc, nu1, nu2, cN) in {"c1": ("c1", "m9", "V", 1, 1, 2), "c3": ("c3", "m7", "V", 1, 1, 2),
                                              "w64": ("c1", "m9", "W", 1, 0, 4)}.items():
    b = workloads.rhs(cfg_id)
    dim, N, _ = workloads.CONFIGS[cfg_id]
    if case == "w64":
        N, b = 64, np.random.default_rng(5).uniform(-1, 1, (63, 63))
    cfg = sp.MgConfig(smoother=sp.named(sm), cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=cN)
    u, rep = sp.solve(sp.Grid(N, torch.as_tensor(b).cuda()), cfg, u0=0)
    out[case] = [rep.iterations, rep.residual_norms, hashlib.sha256(u.values.cpu().numpy().tobytes()).hexdigest()]
print(json.dumps(out))

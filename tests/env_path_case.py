"""Helper for test_gpu_parity.test_alternate_paths_bitwise (run in a subprocess so that the
library reads the SPAIMG_* switches fresh): zero-start solves (CASES), printed as JSON
{case: [iterations, norms, sha256(u)]}."""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from paper_2206_05543_b200 import workloads  # noqa: E402

# case: (rhs: a config id or (dim, N, seed)), smoother, cycle, nu1, nu2, coarsest_N
CASES = {
    "c1": ("c1", "m9", "V", 1, 1, 2),
    "c3": ("c3", "m7", "V", 1, 1, 2),
    "w64": ((2, 64, 5), "m9", "W", 1, 0, 4),
    "c1w": ("c1", "m9", "W", 1, 0, 4),
    "c3w": ("c3", "m7", "W", 1, 0, 4),
    "j2w11": ((2, 128, 6), "jacobi2d", "W", 1, 1, 2),
    "m5v02": ((2, 128, 7), "m5", "V", 0, 2, 4),
    "j3w21": ((3, 32, 8), "jacobi3d", "W", 2, 1, 2),
    # two-sweep marches: pre/post pairs with odd and even totals (level-0 parity plan)
    "m9v33": ((2, 2048, 9), "m9", "V", 3, 3, 2),
    "v9w21": ((2, 1024, 10), "vanka9", "W", 2, 1, 4),
    "m5v12": ((2, 2048, 11), "m5", "V", 1, 2, 2),
}


def case_rhs(src):
    if isinstance(src, str):
        dim, N, _ = workloads.CONFIGS[src]
        return N, workloads.rhs(src)
    dim, N, seed = src
    return N, np.random.default_rng(seed).uniform(-1, 1, (N - 1,) * dim)


if __name__ == "__main__":
    out = {}
    for case, (src, sm, cyc, nu1, nu2, cN) in CASES.items():
        N, b = case_rhs(src)
        cfg = sp.MgConfig(smoother=sp.named(sm), cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=cN)
        u, rep = sp.solve(sp.Grid(N, torch.as_tensor(b).cuda()), cfg, u0=0)
        out[case] = [rep.iterations, rep.residual_norms, hashlib.sha256(u.values.cpu().numpy().tobytes()).hexdigest()]
    print(json.dumps(out))

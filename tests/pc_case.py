"""Helper for test_gpu_parity.test_pc_ragged_vs_oracle (run in a subprocess so that the library
reads SPAIMG_PC2_N / SPAIMG_PC3_N / SPAIMG_FLAT_N* fresh): 2D and 3D cycles with the K3 + K1 march
(prolongation + correction fused into the first post-sweep, multigrid.py:184-185) on EVERY level,
ragged strip / tile edges included, checked bitwise against the C oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from oracle import c_oracle, numpy_oracle as npo  # noqa: E402

# dim, N, smoother, cycle, nu1, nu2, coarsest_N, dtype
CASES = [
    (2, 96, "m9", "V", 1, 1, 3, "float64"),
    (2, 80, "jacobi2d", "V", 1, 2, 5, "float64"),
    (2, 64, "m5", "W", 1, 1, 2, "float64"),
    (2, 1032, "vanka9", "V", 1, 1, 129, "float64"),
    (2, 96, "m9", "V", 1, 1, 3, "float32"),
    (3, 96, "m7", "V", 1, 1, 3, "float64"),
    (3, 80, "jacobi3d", "V", 1, 2, 5, "float64"),
    (3, 64, "m7", "W", 1, 1, 2, "float64"),
    (3, 88, "m7", "V", 0, 1, 11, "float64"),
    (3, 96, "m7", "V", 1, 1, 3, "float32"),
    (3, 72, "jacobi3d", "V", 2, 2, 9, "float32"),
]

if __name__ == "__main__":
    only = int(sys.argv[1]) if len(sys.argv) > 1 else -1
    for i, (dim, N, sm, cyc, nu1, nu2, cN, dtype) in enumerate(CASES):
        if only >= 0 and i != only:
            continue
        npdt = np.float64 if dtype == "float64" else np.float32
        tdt = torch.float64 if dtype == "float64" else torch.float32
        rng = np.random.default_rng(N + nu1)
        x = rng.uniform(-1, 1, (N - 1,) * dim).astype(npdt)
        b = rng.uniform(-1, 1, (N - 1,) * dim).astype(npdt)
        M = sp.named(sm)
        cfg = sp.MgConfig(smoother=M, cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=cN)
        s = sp.Solver(cfg, dim, N, dtype=dtype)
        s.load(torch.as_tensor(b).cuda(), torch.as_tensor(x).cuda())
        s.cycles(2)
        got = torch.empty((N - 1,) * dim, dtype=tdt, device="cuda")
        s.store(got)
        ref = x
        for _ in range(2):
            ref = c_oracle.cycle(ref, b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, nu1, nu2,
                                 2 if cyc == "W" else 1, cN, dtype=npdt)
        assert np.array_equal(got.cpu().numpy(), ref), (dim, N, sm, cyc, nu1, nu2, cN, dtype)
        print("ok", dim, N, sm, cyc, nu1, nu2, cN, dtype, s.stats(), flush=True)
    print("PC OK")

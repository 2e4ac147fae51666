"""Helper for test_gpu_parity.test_pc3_ragged_vs_oracle (run in a subprocess so that the library
reads SPAIMG_PC3_N / SPAIMG_FLAT_N3 fresh): 3D cycles with the K3 + K1 plane march (prolongation +
correction fused into the first post-sweep, multigrid.py:184-185) on EVERY level, ragged tile
edges included, checked bitwise against the C oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from oracle import c_oracle, numpy_oracle as npo  # noqa: E402

# N, smoother, cycle, nu1, nu2, coarsest_N, dtype
CASES = [
    (96, "m7", "V", 1, 1, 3, "float64"),
    (80, "jacobi3d", "V", 1, 2, 5, "float64"),
    (64, "m7", "W", 1, 1, 2, "float64"),
    (88, "m7", "V", 0, 1, 11, "float64"),
    (96, "m7", "V", 1, 1, 3, "float32"),
    (72, "jacobi3d", "V", 2, 2, 9, "float32"),
]

if __name__ == "__main__":
    only = int(sys.argv[1]) if len(sys.argv) > 1 else -1
    for i, (N, sm, cyc, nu1, nu2, cN, dtype) in enumerate(CASES):
        if only >= 0 and i != only:
            continue
        npdt = np.float64 if dtype == "float64" else np.float32
        tdt = torch.float64 if dtype == "float64" else torch.float32
        rng = np.random.default_rng(N + nu1)
        x = rng.uniform(-1, 1, (N - 1,) * 3).astype(npdt)
        b = rng.uniform(-1, 1, (N - 1,) * 3).astype(npdt)
        M = sp.named(sm)
        cfg = sp.MgConfig(smoother=M, cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=cN)
        s = sp.Solver(cfg, 3, N, dtype=dtype)
        s.load(torch.as_tensor(b).cuda(), torch.as_tensor(x).cuda())
        s.cycles(2)
        got = torch.empty((N - 1,) * 3, dtype=tdt, device="cuda")
        s.store(got)
        ref = x
        for _ in range(2):
            ref = c_oracle.cycle(ref, b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, nu1, nu2,
                                 2 if cyc == "W" else 1, cN, dtype=npdt)
        assert np.array_equal(got.cpu().numpy(), ref), (N, sm, cyc, nu1, nu2, cN, dtype)
        print("ok", N, sm, cyc, nu1, nu2, cN, dtype, s.stats(), flush=True)
    print("PC3 OK")

"""Solves beyond BASELINE's sizes, for the record: 2D 16383^2 m9 V(1,1) and 3D 1023^3 m7
V(1,1), seeded U[-1,1] right-hand side, zero start, to 1e-10; one cycle of each checked bitwise
against the C oracle.   python tools/big_solve.py [2d|3d]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from oracle import c_oracle, numpy_oracle as npo  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "2d"
dim, N, sm = (2, 16384, "m9") if which == "2d" else (3, 1024, "m7")
M = sp.named(sm)
rng = np.random.default_rng(0)
b = rng.uniform(-1, 1, (N - 1,) * dim)
cfg = sp.MgConfig(smoother=M, cycle="V", nu1=1, nu2=1, coarsest_N=2, tol=1e-10)
s = sp.Solver(cfg, dim, N)
bd = torch.as_tensor(b).cuda()
s.load(bd)
s.run()
ts = []
for _ in range(3):
    s.load(None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hist, k, conv = s.run()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
t = float(np.median(ts))
st = s.stats()
n = (N - 1) ** dim
print(f"{dim}D N={N} {sm} V(1,1): {k} cycles, converged {conv}, {t:.2f} ms to 1e-10, {t / k:.3f} ms/cycle, "
      f"{n * k / t / 1e6:.1f} G DOF/s, {st['bytes_per_cycle'] / (t / k) / 1e6:.0f} GB/s of the 8d bytes, "
      f"rho_hat {(hist[-1] / hist[0]) ** (1.0 / k):.4f}", flush=True)
# one cycle bitwise against the C oracle
s.load(bd)
s.cycles(1)
got = torch.empty((N - 1,) * dim, dtype=torch.float64, device="cuda")
s.store(got)
t0 = time.time()
ref = c_oracle.cycle(np.zeros_like(b), b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, 1, 1, 1, 2)
print(f"oracle cycle {time.time() - t0:.1f} s; bitwise equal: {np.array_equal(got.cpu().numpy(), ref)}", flush=True)

"""Workload of the sanitizer-substitute tier (tests/test_debug_checks.py, profiles/r02_checked_build.md):
every kernel family of the library on small grids, run against the checked build
(SPAIMG_DEBUG=1: NaN-poisoned buffers, jittered barriers).  compute-sanitizer is closed on the
GPU pool; where it is available, tools/gpu_sanitize.sh runs the same workload under its tools.

    SPAIMG_DEBUG=1 SPAIMG_FLAT_N2=0 SPAIMG_FLAT_N3=0 python tools/sanitize_case.py

With the flat thresholds at 0 the marching kernels (cp.async.bulk / TMA + mbarrier rings, the
fused norm, K1+K3, K2 marches) run on every level; with the defaults the flat tile kernels do.
Both shared-memory coarse engines run: the compile-time one (power-of-two sizes: 2D N=128 enters
at 64, 3D N=32 at 16) and the op-list interpreter (N=96 and N=24, coarse sizes 3 -> warp LU).
Every result is checked bitwise against the C oracle, so a sanitizer run is also a parity run.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from oracle import c_oracle, numpy_oracle as npo  # noqa: E402

rng = np.random.default_rng(99)


def dev(a, dt=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dt)


def check_solve(dim, N, sm, cyc, nu1, nu2, cN, dtype="float64", max_iters=3):
    npdt = np.float64 if dtype == "float64" else np.float32
    tdt = torch.float64 if dtype == "float64" else torch.float32
    b = rng.uniform(-1, 1, (N - 1,) * dim).astype(npdt)
    M = sp.named(sm)
    cfg = sp.MgConfig(smoother=M, cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=cN, max_iters=max_iters, tol=1e-30)
    u, rep = sp.solve(sp.Grid(N, dev(b, tdt)), cfg, u0=0)
    g = 2 if cyc == "W" else 1
    uo, norms, k, conv = c_oracle.solve_history(b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, nu1, nu2, g, cN,
                                                tol=1e-30, max_iters=max_iters, dtype=npdt)
    assert rep.iterations == k, (dim, N, sm, cyc, rep.iterations, k)
    assert np.array_equal(u.values.cpu().numpy(), uo), (dim, N, sm, cyc, nu1, nu2, cN, dtype)
    print("ok solve", dim, N, sm, f"{cyc}({nu1},{nu2})", f"cN={cN}", dtype, flush=True)


def check_operators(dim, N):
    x = rng.uniform(-1, 1, (N - 1,) * dim)
    b = rng.uniform(-1, 1, (N - 1,) * dim)
    e = rng.uniform(-1, 1, (N // 2 - 1,) * dim)
    u, bb = sp.Grid(N, dev(x)), sp.Grid(N, dev(b))
    M = sp.named("m9" if dim == 2 else "m7")
    mt = npo.terms_of(M.stencil)
    assert np.array_equal(sp.smooth(u, bb, M.stencil, M.omega_opt_analytic, 2).values.cpu().numpy(),
                          c_oracle.smooth(x, b, N, mt, M.omega_opt_analytic, 2))
    # a radius-2 smoother: the unfused residual + relaxation kernels
    far = dict(M.stencil.entries)
    from fractions import Fraction
    far[(2,) + (0,) * (dim - 1)] = Fraction(1, 50)
    S2 = sp.Stencil(dim, far, 2)
    assert np.array_equal(sp.smooth(u, bb, S2, 0.1, 2).values.cpu().numpy(),
                          c_oracle.smooth(x, b, N, npo.terms_of(S2), 0.1, 2))
    far[(0,) * (dim - 1) + (-3,)] = Fraction(1, 70)  # radius 3: a three-cell frame on every level
    S3 = sp.Stencil(dim, far, 2)
    assert np.array_equal(sp.smooth(u, bb, S3, 0.1, 2).values.cpu().numpy(),
                          c_oracle.smooth(x, b, N, npo.terms_of(S3), 0.1, 2))
    Nc = 64 if dim == 2 else 16
    xc = rng.uniform(-1, 1, (Nc - 1,) * dim)
    bc = rng.uniform(-1, 1, (Nc - 1,) * dim)
    cfg3 = sp.MgConfig(smoother=S3, omega=0.1, cycle="W", nu1=1, nu2=1, coarsest_N=2)
    assert np.array_equal(sp.cycle(sp.Grid(Nc, dev(xc)), sp.Grid(Nc, dev(bc)), cfg3).values.cpu().numpy(),
                          c_oracle.cycle(xc, bc, Nc, npo.terms_of(S3), 0.1, 1, 1, 2, 2))
    assert np.array_equal(sp.residual_restrict(u, bb).values.cpu().numpy(), c_oracle.residual_restrict(x, b, N))
    assert np.array_equal(sp.prolong_correct(u, sp.Grid(N // 2, dev(e))).values.cpu().numpy(),
                          c_oracle.prolong_correct(x, e))
    sp.restrict(u)
    sp.prolong(sp.Grid(N // 2, dev(e)), N)
    M.stencil.apply  # noqa: B018  (reference API object)
    sp.multigrid.apply_stencil(M.stencil, u)
    assert abs(sp.residual_norm(u, bb) - c_oracle.residual_norm(x, b, N)) <= 1e-12 * c_oracle.residual_norm(x, b, N)
    print("ok operators", dim, N, flush=True)


def main():
    torch.cuda.set_device(0)
    check_operators(2, 66)
    check_operators(3, 18)
    # compile-time engine (power of two) and the fine-level kernels
    check_solve(2, 128, "m9", "V", 1, 1, 2)
    check_solve(2, 128, "m9", "W", 1, 0, 4)
    check_solve(2, 128, "jacobi2d", "V", 2, 2, 4)
    check_solve(2, 128, "m5", "W", 1, 1, 2)
    check_solve(3, 32, "m7", "V", 1, 1, 2)
    check_solve(3, 32, "m7", "W", 1, 0, 4)
    check_solve(3, 32, "jacobi3d", "V", 0, 2, 2)
    check_solve(2, 128, "m9", "V", 1, 1, 2, dtype="float32")
    check_solve(3, 32, "m7", "W", 1, 0, 4, dtype="float32")
    # op-list interpreter (non power-of-two hierarchies, coarse LU on one warp)
    check_solve(2, 96, "m9", "W", 1, 0, 3)
    check_solve(3, 24, "m7", "W", 1, 1, 3)
    # device PCG64 start, pipelined batch
    from paper_2206_05543_b200.multigrid import device_uniform
    like = torch.empty((63, 63), dtype=torch.float64, device="cuda")
    assert np.array_equal(device_uniform(5, like).cpu().numpy(), np.random.default_rng(5).uniform(0, 1, (63, 63)))
    cfg = sp.MgConfig(smoother=sp.named("m9"), cycle="V", nu1=1, nu2=1, coarsest_N=2, max_iters=3, tol=1e-30)
    so = sp.Solver(cfg, 2, 64)
    bs = [rng.uniform(-1, 1, (63, 63)) for _ in range(2)]
    us = [np.empty((63, 63)) for _ in range(2)]
    so.solve_batch(bs, us)
    torch.cuda.synchronize()
    print("ok all", flush=True)


if __name__ == "__main__":
    main()

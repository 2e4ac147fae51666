"""Seeded random configurations of the whole cycle path against the C oracle (bitwise), run by
test_gpu_parity.test_random_configs_vs_oracle in a subprocess: mesh counts with ragged strips /
tiles, every named smoother, V / W, nu1, nu2 in 0..2, coarsest_N from the halving chain, fp64 and
fp32, and random settings of the path switches (flat / marching thresholds, K3 + K1 thresholds,
engine entry, two-sweep marches), which the library reads when a solver is planned."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_05543_b200 as sp  # noqa: E402
from oracle import c_oracle, numpy_oracle as npo  # noqa: E402

SWITCHES = {
    "SPAIMG_FLAT_N2": ["0", "64", None], "SPAIMG_FLAT_N3": ["0", "16", None],
    "SPAIMG_PC2_N": ["0", "1", None], "SPAIMG_PC3_N": ["0", "1", None],
    "SPAIMG_TAIL_N": ["0", "8", "32", None], "SPAIMG_SWEEP2": ["0", None], "SPAIMG_TAIL_FAST": ["0", None],
}


def chain(N):
    """mesh counts reachable by halving N (each a valid coarsest_N)"""
    out = [N]
    while out[-1] % 2 == 0 and out[-1] // 2 >= 2:
        out.append(out[-1] // 2)
    return out


def main(seed, ncases):
    rng = np.random.default_rng(seed)
    for case in range(ncases):
        dim = int(rng.choice([2, 3]))
        if dim == 2:
            N = int(rng.choice([24, 40, 48, 96, 132, 160, 192, 320, 384, 640, 1280, 1536, 2304]))
        else:
            N = int(rng.choice([12, 20, 24, 40, 48, 72, 80, 96, 144, 160]))
        ch = chain(N)
        # keep the coarse LU small (n^dim unknowns)
        cands = [c for c in ch[1:] if (c - 1) ** dim <= 1500]
        if not cands:
            continue
        cN = int(rng.choice(cands))
        sm = str(rng.choice([k for k in sp.NAMED_SMOOTHER_IDS if sp.named(k).dim == dim]))
        cyc = str(rng.choice(["V", "W"]))
        nu1, nu2 = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        if nu1 + nu2 == 0:
            nu1 = 1
        dtype = str(rng.choice(["float64", "float64", "float32"]))
        env = {}
        for k, vals in SWITCHES.items():
            v = vals[int(rng.integers(0, len(vals)))]
            os.environ.pop(k, None)
            if v is not None:
                os.environ[k] = v
                env[k[7:]] = v
        # W-cycles visit 2^depth coarse levels: keep them shallow
        if cyc == "W" and len(ch) - ch.index(cN) > 0 and (N // cN) > 64:
            cyc = "V"
        npdt = np.float64 if dtype == "float64" else np.float32
        tdt = torch.float64 if dtype == "float64" else torch.float32
        x = rng.uniform(-1, 1, (N - 1,) * dim).astype(npdt)
        b = rng.uniform(-1, 1, (N - 1,) * dim).astype(npdt)
        M = sp.named(sm)
        cfg = sp.MgConfig(smoother=M, cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=cN)
        print("case", case, dim, N, sm, f"{cyc}({nu1},{nu2})", f"cN={cN}", dtype, env, flush=True)
        s = sp.Solver(cfg, dim, N, dtype=dtype)
        s.load(torch.as_tensor(b).cuda(), torch.as_tensor(x).cuda())
        s.cycles(2)
        got = torch.empty((N - 1,) * dim, dtype=tdt, device="cuda")
        s.store(got)
        ref = x
        for _ in range(2):
            ref = c_oracle.cycle(ref, b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, nu1, nu2,
                                 2 if cyc == "W" else 1, cN, dtype=npdt)
        ok = np.array_equal(got.cpu().numpy(), ref)
        assert ok, "MISMATCH"
        del s
    print("FUZZ OK")


def operators(seed, ncases):
    """The per-operator entry points (smooth with 0..3 steps incl. odd mesh counts, residual +
    restriction, prolongation + correction, residual norm) at random sizes, host and device
    arrays, fp64 and fp32, bitwise against the C oracle."""
    rng = np.random.default_rng(1000 + seed)
    for case in range(ncases):
        dim = int(rng.choice([2, 3]))
        N = int(rng.integers(3, 700)) if dim == 2 else int(rng.integers(3, 90))
        dtype = str(rng.choice(["float64", "float32"]))
        side = str(rng.choice(["host", "device"]))
        if side == "host":
            dtype = "float64"  # host grids are float64 like the reference's (grids.py:24)
        npdt = np.float64 if dtype == "float64" else np.float32
        tdt = torch.float64 if dtype == "float64" else torch.float32
        sm = str(rng.choice([k for k in sp.NAMED_SMOOTHER_IDS if sp.named(k).dim == dim]))
        M = sp.named(sm)
        mt = npo.terms_of(M.stencil)
        steps = int(rng.integers(0, 4))
        x = rng.uniform(-1, 1, (N - 1,) * dim).astype(npdt)
        b = rng.uniform(-1, 1, (N - 1,) * dim).astype(npdt)
        wrap = (lambda a: a) if side == "host" else (lambda a: torch.as_tensor(a).to("cuda", tdt))
        host = lambda g: g.values.cpu().numpy() if torch.is_tensor(g.values) else g.values  # noqa: E731
        print("op case", case, dim, N, sm, steps, dtype, side, flush=True)
        u, bb = sp.Grid(N, wrap(x)), sp.Grid(N, wrap(b))
        got = host(sp.smooth(u, bb, M.stencil, M.omega_opt_analytic, steps))
        assert np.array_equal(got, c_oracle.smooth(x, b, N, mt, M.omega_opt_analytic, steps, dtype=npdt)), "smooth"
        assert sp.residual_norm(u, bb) == __import__("pytest").approx(c_oracle.residual_norm(x, b, N, dtype=npdt), rel=1e-12)
        if N % 2 == 0 and N >= 4:
            e = rng.uniform(-1, 1, (N // 2 - 1,) * dim).astype(npdt)
            assert np.array_equal(host(sp.residual_restrict(u, bb)), c_oracle.residual_restrict(x, b, N, dtype=npdt)), "rr"
            assert np.array_equal(host(sp.prolong_correct(u, sp.Grid(N // 2, wrap(e)))),
                                  c_oracle.prolong_correct(x, e, dtype=npdt)), "pc"
    print("FUZZ OK")


if __name__ == "__main__":
    if len(sys.argv) > 3 and sys.argv[3] == "ops":
        operators(int(sys.argv[1]), int(sys.argv[2]))
        sys.exit(0)
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 0, int(sys.argv[2]) if len(sys.argv) > 2 else 24)

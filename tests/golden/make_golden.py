"""Generate the committed golden fixtures by running the REFERENCE `spaimg`.

This script is the only place that imports the reference package.  It
needs `/root/reference/pkg/src` (read-only, present in the build container,
absent on the GPU box), so the fixtures it writes are committed and the
tests only ever read them.

    python tests/golden/make_golden.py ops          # small per-operator / cycle fixtures
    python tests/golden/make_golden.py hist c1 c3   # residual histories (zero u0)
    python tests/golden/make_golden.py hist c2      # ~5 min of CPU
    python tests/golden/make_golden.py hist c4      # ~1 h of CPU, ~10 GB RSS
    python tests/golden/make_golden.py hist c1 c3 c2 --only "W("   # the W(1,0) defaults only

The zero-u0 history loop below is the harness SURVEY.md Finding 2 describes:
it calls the reference `cycle()` and repeats `solve()`'s norm and stop logic
(reference `pkg/src/spaimg/multigrid.py:206-219`) with u0 = 0 instead of the
seeded U(0,1) start of `multigrid.py:204-205`.
"""

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF_SRC = os.environ.get("SPAIMG_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)

import spaimg  # noqa: E402  (the reference)
from spaimg import (Grid, MgConfig, cycle, laplacian, named, prolong,  # noqa: E402
                    restrict, smooth, tee, upsilon)
from spaimg.problems import Problem, assemble_rhs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


# ----------------------------------------------------------------------------
# configs (BASELINE.json lines 7-11)
# ----------------------------------------------------------------------------

def rhs_for(cfg_id: str) -> Grid:
    if cfg_id == "c1":
        p = Problem(dim=2, f=lambda x, y: 2 * math.pi ** 2 * np.sin(math.pi * x) * np.sin(math.pi * y))
        return assemble_rhs(p, 256)
    if cfg_id == "c3":
        p = Problem(dim=3, f=lambda x, y, z: 3 * math.pi ** 2 * np.sin(math.pi * x)
                    * np.sin(math.pi * y) * np.sin(math.pi * z))
        return assemble_rhs(p, 128)
    if cfg_id == "c2":
        return Grid(4096, np.random.default_rng(0).uniform(-1, 1, (4095, 4095)))
    if cfg_id == "c4":
        return Grid(512, np.random.default_rng(1).uniform(-1, 1, (511, 511, 511)))
    raise KeyError(cfg_id)


# (smoother, nu1, nu2[, cycle, coarsest_N]); the 3-tuples are V-cycles with coarsest_N = 2.
# The W(1,0), coarsest_N = 4 runs are the reference MgConfig defaults (multigrid.py:39-43).
RUNS = {
    "c1": [("m9", 1, 1), ("m9", 1, 0, "W", 4)],
    "c3": [("m7", 1, 1), ("m7", 1, 0, "W", 4)],
    "c2": [("m9", 1, 1), ("m9", 2, 2), ("jacobi2d", 1, 1), ("jacobi2d", 2, 2), ("m9", 1, 0, "W", 4)],
    "c4": [("m7", 1, 1), ("m7", 2, 2), ("jacobi3d", 1, 1), ("jacobi3d", 2, 2), ("m7", 1, 0, "W", 4)],
}


def run_key(cid, run):
    sm, nu1, nu2 = run[:3]
    cyc, nc = (run[3], run[4]) if len(run) > 3 else ("V", 2)
    key = f"{cid}/{sm}/{cyc}({nu1},{nu2})"
    return (key if (cyc, nc) == ("V", 2) else f"{key}/cN{nc}"), sm, nu1, nu2, cyc, nc


def zero_start_history(b: Grid, cfg: MgConfig):
    """Zero-u0 twin of reference solve(): multigrid.py:206-219 with u0 = 0."""
    A = laplacian(b.dim)
    u = Grid.zeros(b.dim, b.N)
    norms = [float(np.linalg.norm(b.values - A.apply(u).values))]
    shas = []
    k = 0
    converged = False
    t0 = time.perf_counter()
    while k < cfg.max_iters:
        u = cycle(u, b, cfg)
        k += 1
        if k == 1:
            shas.append(sha(u.values))
        norms.append(float(np.linalg.norm(b.values - A.apply(u).values)))
        if norms[-1] <= cfg.tol * norms[0]:
            converged = True
            break
    wall = time.perf_counter() - t0
    return u, dict(norms=norms, iterations=k, converged=converged,
                   rho_hat=(norms[-1] / norms[0]) ** (1.0 / k),
                   sha_u_cycle1=shas[0], sha_u_final=sha(u.values),
                   s_per_cycle=wall / k, wall_s=wall)


def cmd_hist(cfg_ids, only=None):
    path = os.path.join(HERE, "histories.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for cid in cfg_ids:
        b = rhs_for(cid)
        for run in RUNS[cid]:
            key, sm, nu1, nu2, cyc, nc = run_key(cid, run)
            if only and only not in key:
                continue
            cfg = MgConfig(smoother=named(sm), cycle=cyc, nu1=nu1, nu2=nu2,
                           coarsest_N=nc, tol=1e-10, max_iters=100)
            _, rec = zero_start_history(b, cfg)
            rec.update(config=cid, smoother=sm, nu1=nu1, nu2=nu2, cycle=cyc,
                       coarsest_N=nc, tol=1e-10, N=b.N, dim=b.dim, sha_b=sha(b.values),
                       host_cpu=_cpu_model(), numpy=np.__version__)
            data[key] = rec
            print(key, rec["iterations"], rec["norms"][-1], f"{rec['s_per_cycle']:.3f} s/cycle",
                  flush=True)
            # re-read + merge so parallel invocations do not clobber each other
            cur = json.load(open(path)) if os.path.exists(path) else {}
            cur[key] = rec
            with open(path, "w") as f:
                json.dump(cur, f, indent=1, sort_keys=True)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "?"


# ----------------------------------------------------------------------------
# small per-operator and per-cycle fixtures
# ----------------------------------------------------------------------------

def custom_smoothers(dim):
    # custom stencils exercise non-named term lists (and a zero centre kept by upsilon)
    if dim == 2:
        return {"ups_1_2_3": (upsilon(1, 2, 3), 0.05), "ups_0_1_0": (upsilon(0, 1, 0), 0.1)}
    return {"tee_3_1": (tee(3, 1), 0.2)}


def cmd_ops():
    out = {}
    meta = {"generator": "tests/golden/make_golden.py ops", "reference": REF_SRC,
            "spaimg_version": spaimg.__version__, "numpy": np.__version__}
    rng = np.random.default_rng(20240601)
    for dim, Ns in ((2, (4, 8, 12, 16, 34)), (3, (4, 8, 12))):
        smoothers = {k: (named(k).stencil, named(k).omega_opt_analytic)
                     for k in spaimg.NAMED_SMOOTHER_IDS if named(k).dim == dim}
        smoothers.update(custom_smoothers(dim))
        for N in Ns:
            shape = (N - 1,) * dim
            x = rng.uniform(-1, 1, shape)
            b = rng.uniform(-1, 1, shape)
            tag = f"d{dim}_N{N}"
            out[f"{tag}/x"] = x
            out[f"{tag}/b"] = b
            u, bb = Grid(N, x), Grid(N, b)
            out[f"{tag}/apply/A"] = laplacian(dim).apply(u).values
            for name, (M, om) in smoothers.items():
                out[f"{tag}/apply/{name}"] = M.apply(u).values
                out[f"{tag}/smooth1/{name}"] = smooth(u, bb, M, om, 1).values
                out[f"{tag}/smooth2/{name}"] = smooth(u, bb, M, om, 2).values
                out[f"{tag}/omega/{name}"] = np.array(om)
            if N % 2 == 0 and N // 2 >= 2:
                r = b - laplacian(dim).apply(u).values
                out[f"{tag}/restrict_r"] = restrict(Grid(N, r)).values
                e = rng.uniform(-1, 1, (N // 2 - 1,) * dim)
                out[f"{tag}/e"] = e
                out[f"{tag}/prolong_e"] = prolong(Grid(N // 2, e), N).values
                out[f"{tag}/prolong_correct"] = x + prolong(Grid(N // 2, e), N).values
    # whole cycles: V/W, coarsest_N 2/4, a few smoothers, random start
    cyc_cases = [
        (2, 32, "m9", "V", 1, 1, 2), (2, 32, "m9", "W", 1, 0, 4), (2, 32, "jacobi2d", "V", 2, 2, 2),
        (2, 16, "vanka9", "W", 1, 1, 2), (2, 24, "m9", "V", 1, 1, 3), (2, 32, "m5", "V", 0, 2, 4),
        (3, 16, "m7", "V", 1, 1, 2), (3, 16, "m7", "W", 1, 0, 4), (3, 16, "jacobi3d", "V", 2, 1, 2),
        (3, 16, "m7", "V", 1, 1, 4),
    ]
    for dim, N, sm, cyc, nu1, nu2, nc in cyc_cases:
        shape = (N - 1,) * dim
        x = rng.uniform(-1, 1, shape)
        b = rng.uniform(-1, 1, shape)
        cfg = MgConfig(smoother=named(sm), cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=nc)
        tag = f"cycle/d{dim}_N{N}_{sm}_{cyc}{nu1}{nu2}_c{nc}"
        out[f"{tag}/x"] = x
        out[f"{tag}/b"] = b
        out[f"{tag}/out"] = cycle(Grid(N, x), Grid(N, b), cfg).values
    np.savez_compressed(os.path.join(HERE, "ops_golden.npz"), **out)

    # default solve() path (seeded U(0,1) start, multigrid.py:188-227) on small problems
    solves = {}
    for dim, N, sm, cyc, nu1, nu2, nc, seed in [
        (2, 64, "m9", "W", 1, 0, 4, 0), (2, 64, "m9", "V", 1, 1, 2, 0), (2, 32, "jacobi2d", "V", 1, 1, 4, 3),
        (3, 16, "m7", "V", 1, 1, 2, 0), (3, 16, "m7", "W", 1, 0, 4, 1),
    ]:
        b = Grid(N, np.random.default_rng(100 + N + dim).uniform(-1, 1, (N - 1,) * dim))
        cfg = MgConfig(smoother=named(sm), cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=nc, rng_seed=seed)
        u, rep = spaimg.solve(b, cfg)
        solves[f"d{dim}_N{N}_{sm}_{cyc}{nu1}{nu2}_c{nc}_s{seed}"] = dict(
            dim=dim, N=N, smoother=sm, cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=nc, rng_seed=seed,
            b_seed=100 + N + dim, norms=rep.residual_norms, iterations=rep.iterations,
            converged=rep.converged, rho_hat=rep.rho_hat, sha_u=sha(u.values))
    meta["solves"] = solves
    with open(os.path.join(HERE, "ops_meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays,", len(solves), "solves")


if __name__ == "__main__":
    if sys.argv[1] == "ops":
        cmd_ops()
    elif sys.argv[1] == "hist":
        # optional trailing "--only <substring>" selects runs by key, e.g. --only W(
        args = sys.argv[2:]
        only = None
        if "--only" in args:
            i = args.index("--only")
            only = args[i + 1]
            args = args[:i] + args[i + 2:]
        cmd_hist(args, only)
    else:
        raise SystemExit(__doc__)

"""GPU parity of the sm_100a hot path against the reference's golden vectors and the oracle.

float64: bitwise (np.array_equal) per operator and per cycle; residual histories
within 1e-8 relative with identical cycle counts (north star, BASELINE.json:5).
float32: bitwise against the float32 restatement.
"""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2206_05543_b200 as sp  # noqa: E402
from oracle import c_oracle, numpy_oracle as npo  # noqa: E402
from paper_2206_05543_b200 import workloads  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [(2, N) for N in (4, 8, 12, 16, 34)] + [(3, N) for N in (4, 8, 12)]


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")


def smoothers_for(dim):
    out = {k: (sp.named(k).stencil, sp.named(k).omega_opt_analytic)
           for k in sp.NAMED_SMOOTHER_IDS if sp.named(k).dim == dim}
    if dim == 2:
        out["ups_1_2_3"] = (sp.upsilon(1, 2, 3), 0.05)
        out["ups_0_1_0"] = (sp.upsilon(0, 1, 0), 0.1)
    else:
        out["tee_3_1"] = (sp.tee(3, 1), 0.2)
    return out


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to("cuda", dtype)


def host(t):
    return t.values.cpu().numpy() if torch.is_tensor(t.values) else t.values


@pytest.mark.parametrize("side", ["host", "device"])
@pytest.mark.parametrize("dim,N", CASES)
def test_operators_vs_reference_golden(golden_ops, side, dim, N):
    g = golden_ops
    t = f"d{dim}_N{N}"
    x, b = g[t + "/x"], g[t + "/b"]
    wrap = (lambda a: a) if side == "host" else dev
    u, bb = sp.Grid(N, wrap(x)), sp.Grid(N, wrap(b))
    for name, (M, om) in smoothers_for(dim).items():
        for steps in (1, 2):
            got = host(sp.smooth(u, bb, M, om, steps))
            assert np.array_equal(got, g[f"{t}/smooth{steps}/{name}"]), (name, steps)
        assert np.array_equal(host(M.apply(u)), g[f"{t}/apply/{name}"]), name
    assert np.array_equal(host(sp.laplacian(dim).apply(u)), g[f"{t}/apply/A"])
    assert np.array_equal(host(sp.smooth(u, bb, sp.named("m9" if dim == 2 else "m7").stencil, 0.3, 0)), x)
    if f"{t}/restrict_r" in g:
        assert np.array_equal(host(sp.residual_restrict(u, bb)), g[t + "/restrict_r"])
        r = b - g[f"{t}/apply/A"]
        assert np.array_equal(host(sp.restrict(sp.Grid(N, wrap(r)))), g[t + "/restrict_r"])
        e = sp.Grid(N // 2, wrap(g[t + "/e"]))
        assert np.array_equal(host(sp.prolong(e, N)), g[t + "/prolong_e"])
        assert np.array_equal(host(sp.prolong_correct(u, e)), g[t + "/prolong_correct"])


def _cycle_cases(g):
    for k in g.keys():
        if k.startswith("cycle/") and k.endswith("/out"):
            tag = k[:-4]
            d, N, sm, cyc, c = tag.split("/")[1].split("_")
            yield tag, int(d[1:]), int(N[1:]), sm, cyc[0], int(cyc[1]), int(cyc[2]), int(c[1:])


@pytest.mark.parametrize("side", ["host", "device"])
def test_cycles_vs_reference_golden(golden_ops, side):
    wrap = (lambda a: a) if side == "host" else dev
    n = 0
    for tag, dim, N, sm, cyc, nu1, nu2, nc in _cycle_cases(golden_ops):
        cfg = sp.MgConfig(smoother=sp.named(sm), cycle=cyc, nu1=nu1, nu2=nu2, coarsest_N=nc)
        out = sp.cycle(sp.Grid(N, wrap(golden_ops[tag + "/x"])), sp.Grid(N, wrap(golden_ops[tag + "/b"])), cfg)
        assert np.array_equal(host(out), golden_ops[tag + "/out"]), tag
        n += 1
    assert n >= 10


@pytest.mark.parametrize("side", ["host", "device"])
def test_default_solve_vs_reference_golden(golden_meta, side):
    """solve() with the reference's seeded U(0,1) start (multigrid.py:204-205); device grids draw
    it on the GPU (spaimg_fill_uniform), host grids with numpy."""
    for key, rec in golden_meta["solves"].items():
        dim, N = rec["dim"], rec["N"]
        b = np.random.default_rng(rec["b_seed"]).uniform(-1, 1, (N - 1,) * dim)
        cfg = sp.MgConfig(smoother=sp.named(rec["smoother"]), cycle=rec["cycle"], nu1=rec["nu1"], nu2=rec["nu2"],
                          coarsest_N=rec["coarsest_N"], rng_seed=rec["rng_seed"])
        u, rep = sp.solve(sp.Grid(N, b if side == "host" else dev(b)), cfg)
        u = sp.Grid(N, host(u))
        assert rep.iterations == rec["iterations"] and rep.converged == rec["converged"], key
        rel = max(abs(a - r) / r for a, r in zip(rep.residual_norms, rec["norms"]))
        assert rel < 1e-8, (key, rel)
        assert hashlib.sha256(np.ascontiguousarray(u.values).tobytes()).hexdigest() == rec["sha_u"], key
        assert rep.rho_hat == pytest.approx(rec["rho_hat"], rel=1e-8)


def _zero_start(cfg_id, sm, nu1, nu2, side="device", cycle="V", coarsest_N=2):
    b = workloads.rhs(cfg_id)
    dim, N, _ = workloads.CONFIGS[cfg_id]
    cfg = sp.MgConfig(smoother=sp.named(sm), cycle=cycle, nu1=nu1, nu2=nu2, coarsest_N=coarsest_N)
    bg = sp.Grid(N, dev(b) if side == "device" else b)
    u, rep = sp.solve(bg, cfg, u0=0)
    return b, u, rep


@pytest.mark.parametrize("cfg_id,sm", [("c1", "m9"), ("c3", "m7")])
def test_small_configs_histories(golden_hist, cfg_id, sm):
    """Configs 1 and 3 in full: vs the reference golden (when the RHS is bitwise the
    golden one) and always vs the C oracle run here on the same inputs."""
    b, u, rep = _zero_start(cfg_id, sm, 1, 1)
    dim, N, _ = workloads.CONFIGS[cfg_id]
    mt = npo.terms_of(sp.named(sm).stencil)
    uo, norms, k, conv = c_oracle.solve_history(b, N, mt, sp.named(sm).omega_opt_analytic, 1, 1, 1, 2)
    assert rep.iterations == k and rep.converged and conv
    assert max(abs(a - r) / r for a, r in zip(rep.residual_norms, norms)) < 1e-8
    assert np.array_equal(host(u), uo)
    rec = golden_hist[f"{cfg_id}/{sm}/V(1,1)"]
    if hashlib.sha256(b.tobytes()).hexdigest() == rec["sha_b"]:
        assert rep.iterations == rec["iterations"]
        assert max(abs(a - r) / r for a, r in zip(rep.residual_norms, rec["norms"])) < 1e-8
        assert hashlib.sha256(host(u).tobytes()).hexdigest() == rec["sha_u_final"]


@pytest.mark.parametrize("key", ["c2/m9/V(1,1)", "c2/m9/V(2,2)", "c2/jacobi2d/V(1,1)", "c2/jacobi2d/V(2,2)",
                                 "c4/m7/V(1,1)", "c4/m7/V(2,2)", "c4/jacobi3d/V(1,1)", "c4/jacobi3d/V(2,2)",
                                 "c1/m9/W(1,0)/cN4", "c3/m7/W(1,0)/cN4", "c2/m9/W(1,0)/cN4", "c4/m7/W(1,0)/cN4"])
def test_large_configs_vs_reference_golden(golden_hist, key):
    """Configs 1-4 at full size against the reference's own histories (generated in the build
    container, tests/golden/histories.json): identical cycle counts, histories within 1e-8
    relative, and the final iterate bitwise (sha256).  The W(1,0), coarsest_N = 4 runs are the
    reference MgConfig defaults (multigrid.py:39-43)."""
    if key not in golden_hist:
        pytest.skip(f"golden history {key} not generated yet")
    rec = golden_hist[key]
    cfg_id, sm, v = key.split("/")[:3]
    nu1, nu2 = int(v[2]), int(v[4])
    b, u, rep = _zero_start(cfg_id, sm, nu1, nu2, cycle=rec["cycle"], coarsest_N=rec["coarsest_N"])
    assert hashlib.sha256(b.tobytes()).hexdigest() == rec["sha_b"]
    assert rep.iterations == rec["iterations"] and rep.converged
    rel = max(abs(a - r) / r for a, r in zip(rep.residual_norms, rec["norms"]))
    assert rel < 1e-8, rel
    assert hashlib.sha256(host(u).tobytes()).hexdigest() == rec["sha_u_final"]


@pytest.mark.parametrize("dim,N,sm", [(2, 512, "m9"), (2, 256, "jacobi2d"), (2, 130, "vanka9"), (3, 64, "m7"),
                                      (3, 34, "jacobi3d"), (2, 2050, "jacobi2d"), (2, 2048, "m5")])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_medium_operators_vs_oracle(dim, N, sm, dtype):
    """Larger, ragged sizes (N-1 odd, tiles partially filled) vs the C oracle, bitwise."""
    rng = np.random.default_rng(N + dim)
    x = rng.uniform(-1, 1, (N - 1,) * dim)
    b = rng.uniform(-1, 1, (N - 1,) * dim)
    e = rng.uniform(-1, 1, (N // 2 - 1,) * dim)
    npdt = np.float64 if dtype == "float64" else np.float32
    tdt = torch.float64 if dtype == "float64" else torch.float32
    M = sp.named(sm)
    mt = npo.terms_of(M.stencil)
    u, bb = sp.Grid(N, dev(x, tdt)), sp.Grid(N, dev(b, tdt))
    # 2 and 3 steps: pairs of steps run as one two-sweep march on the 2D marching sizes (N > 1024)
    for steps in (2, 3):
        got = host(sp.smooth(u, bb, M.stencil, M.omega_opt_analytic, steps))
        assert got.dtype == npdt
        assert np.array_equal(got, c_oracle.smooth(x, b, N, mt, M.omega_opt_analytic, steps, dtype=npdt)), steps
    assert np.array_equal(host(sp.residual_restrict(u, bb)), c_oracle.residual_restrict(x, b, N, dtype=npdt))
    assert np.array_equal(host(sp.prolong_correct(u, sp.Grid(N // 2, dev(e, tdt)))),
                          c_oracle.prolong_correct(x, e, dtype=npdt))
    nrm = sp.residual_norm(u, bb)
    assert nrm == pytest.approx(c_oracle.residual_norm(x, b, N, dtype=npdt), rel=1e-12)


def test_full_size_properties_2d():
    """Size-independent properties at BASELINE size 4096^2: full weighting of ones is one,
    the restriction/prolongation adjoint relation, determinism."""
    N = 4096
    ones = sp.Grid(N, torch.ones((N - 1, N - 1), dtype=torch.float64, device="cuda"))
    rc = sp.restrict(ones).values
    assert torch.all(rc == 1.0)
    rng = np.random.default_rng(3)
    c = sp.Grid(N // 2, dev(rng.uniform(-1, 1, (N // 2 - 1,) * 2)))
    f = sp.Grid(N, dev(rng.uniform(-1, 1, (N - 1,) * 2)))
    lhs = float((sp.prolong(c, N).values * f.values).sum())
    rhs = 4.0 * float((c.values * sp.restrict(f).values).sum())
    assert lhs == pytest.approx(rhs, rel=1e-12)
    b = workloads.rhs("c2")
    cfg = sp.MgConfig(smoother=sp.named("m9"), cycle="V", nu1=1, nu2=1, coarsest_N=2, max_iters=2)
    u1, r1 = sp.solve(sp.Grid(N, dev(b)), cfg, u0=0)
    u2, r2 = sp.solve(sp.Grid(N, dev(b)), cfg, u0=0)
    assert r1.residual_norms == r2.residual_norms
    assert torch.equal(u1.values, u2.values)


def _custom_stencils(dim):
    """Radius-1 stencils that hit the generic (runtime term list) kernels: a reversed-order
    copy of the paper's smoother and a full box with distinct coefficients."""
    from fractions import Fraction
    base = sp.named("m9" if dim == 2 else "m7").stencil
    rev = sp.Stencil(dim, dict(reversed(list(base.entries.items()))), base.h_exponent)
    import itertools
    box = {}
    for k, o in enumerate(itertools.product((0, 1, -1), repeat=dim)):
        box[o] = Fraction(1, 7 + k) if any(o) else Fraction(3, 4)
    # radius 2 (the unfused residual + relax path, and a 2-cell frame in the tail)
    far = {o: c for o, c in base.entries.items()}
    far[(2,) + (0,) * (dim - 1)] = Fraction(1, 50)
    far[(0,) * (dim - 1) + (-2,)] = Fraction(1, 40)
    # radius 3: a wider zero frame on every level (the reference applies any reach, stencils.py:145-146)
    far3 = dict(far)
    far3[(-3,) + (0,) * (dim - 1)] = Fraction(1, 60)
    far3[(0,) * (dim - 1) + (3,)] = Fraction(1, 70)
    return {"reversed": (rev, 0.15), "box": (sp.Stencil(dim, box, 2), 0.05), "radius2": (sp.Stencil(dim, far, 2), 0.1),
            "radius3": (sp.Stencil(dim, far3, 2), 0.08)}


@pytest.mark.parametrize("dim,N", [(2, 66), (3, 34)])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_generic_stencils_vs_oracle(dim, N, dtype):
    rng = np.random.default_rng(7 * N + dim)
    x = rng.uniform(-1, 1, (N - 1,) * dim)
    b = rng.uniform(-1, 1, (N - 1,) * dim)
    npdt = np.float64 if dtype == "float64" else np.float32
    tdt = torch.float64 if dtype == "float64" else torch.float32
    u, bb = sp.Grid(N, dev(x, tdt)), sp.Grid(N, dev(b, tdt))
    for name, (M, om) in _custom_stencils(dim).items():
        mt = npo.terms_of(M)
        got = host(sp.smooth(u, bb, M, om, 3))
        assert np.array_equal(got, c_oracle.smooth(x, b, N, mt, om, 3, dtype=npdt)), name
        if dtype == "float64":
            Nc = 64 if dim == 2 else 32
            xc = rng.uniform(-1, 1, (Nc - 1,) * dim)
            bc = rng.uniform(-1, 1, (Nc - 1,) * dim)
            for cyc, g in (("V", 1), ("W", 2)):
                cfg = sp.MgConfig(smoother=M, omega=om, cycle=cyc, nu1=1, nu2=1, coarsest_N=2)
                got = host(sp.cycle(sp.Grid(Nc, dev(xc)), sp.Grid(Nc, dev(bc)), cfg))
                assert np.array_equal(got, c_oracle.cycle(xc, bc, Nc, mt, om, 1, 1, g, 2)), (name, cyc)


@pytest.mark.parametrize("dim,N,sm", [(2, 256, "m9"), (3, 32, "m7")])
def test_solve_batch_pipelined_matches_single_solves(dim, N, sm):
    """Solver.solve_batch (host buffers, copies overlapped with the solves) gives, for every
    right-hand side, the same history and bitwise the same iterate as one solve at a time."""
    cfg = sp.MgConfig(smoother=sp.named(sm), cycle="V", nu1=1, nu2=1, coarsest_N=2, tol=1e-10)
    rng = np.random.default_rng(11)
    bs = [torch.as_tensor(rng.uniform(-1, 1, (N - 1,) * dim)).pin_memory() for _ in range(3)]
    us = [torch.empty_like(b).pin_memory() for b in bs]
    solver = sp.Solver(cfg, dim, N)
    res = solver.solve_batch([b.numpy() for b in bs], [u.numpy() for u in us])
    for b, u, (hist, k, conv) in zip(bs, us, res):
        ref_u, rep = sp.solve(sp.Grid(N, b.numpy().copy()), cfg, u0=0)
        assert k == rep.iterations and conv == rep.converged
        assert hist == rep.residual_norms
        assert np.array_equal(u.numpy(), ref_u.values)


@pytest.mark.parametrize("env", [{}, {"SPAIMG_NO_GRAPH": "1"}, {"SPAIMG_TAIL_FAST": "0"}, {"SPAIMG_TAIL_N": "0"}, {"SPAIMG_TAIL_N": "8"},
                                 {"SPAIMG_TAIL_N": "32"}, {"SPAIMG_FLAT_N2": "0", "SPAIMG_FLAT_N3": "0"}],
                         ids=lambda e: ",".join(f"{k[7:]}={v}" for k, v in e.items()) or "default")
def test_alternate_paths_bitwise(env):
    """The default schedule and every tuning switch (eager launches; the shared-memory coarse
    engine off or entered at other sizes; marching kernels on every level) give the same
    iterations, histories and bitwise iterates as the C oracle, over V and W cycles, nu1 = 0,
    coarsest_N 2 and 4, and the C1 / STAR5 / BOX9 / STAR7 smoother shapes (tests/env_path_case.py)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tests"))
    import env_path_case as epc
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "env_path_case.py")], capture_output=True,
                       text=True, timeout=900, env=dict(os.environ, **env))
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    for case, (src, sm, cyc, nu1, nu2, cN) in epc.CASES.items():
        N, b = epc.case_rhs(src)
        M = sp.named(sm)
        uo, norms, k, conv = c_oracle.solve_history(b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, nu1, nu2,
                                                    2 if cyc == "W" else 1, cN)
        it, hist, sha = got[case]
        assert it == k, (case, it, k)
        assert max(abs(a - r) / r for a, r in zip(hist, norms)) < 1e-8, case
        assert sha == hashlib.sha256(uo.tobytes()).hexdigest(), case


@pytest.mark.parametrize("env", [{"SPAIMG_PC3_N": "1", "SPAIMG_PC2_N": "1", "SPAIMG_FLAT_N3": "0", "SPAIMG_FLAT_N2": "0"},
                                 {"SPAIMG_PC3_N": "1", "SPAIMG_PC2_N": "1", "SPAIMG_NO_GRAPH": "1"},
                                 {"SPAIMG_PC3_N": "0", "SPAIMG_PC2_N": "0"}],
                         ids=lambda e: ",".join(f"{k[7:]}={v}" for k, v in e.items()))
def test_pc_ragged_vs_oracle(env):
    """The K3 + K1 marches (prolongation + correction fused into the first post-sweep; 2D row
    march, 3D plane march) on every level the switches allow -- ragged strip / tile edges, boundary
    tiles, odd chunk lengths, fp64 and fp32, every named shape -- bitwise against the C oracle;
    SPAIMG_PC*_N=0 is the unfused K3 then K1."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "pc_case.py")], capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, **env))
    assert r.returncode == 0 and "PC OK" in r.stdout, (r.stdout[-2000:], r.stderr[-3000:])


@pytest.mark.parametrize("dim,N,sm", [(2, 256, "m9"), (2, 4096, "m9"), (2, 512, "jacobi2d"), (3, 64, "m7"),
                                      (3, 256, "m7")])
def test_fp32_cycles_vs_oracle(dim, N, sm):
    """fp32 V(1,1) cycles (marching, K3-fused, flat and tail kernels in float32) bitwise against
    the float32 restatement."""
    rng = np.random.default_rng(3 * N + dim)
    x = rng.uniform(-1, 1, (N - 1,) * dim).astype(np.float32)
    b = rng.uniform(-1, 1, (N - 1,) * dim).astype(np.float32)
    M = sp.named(sm)
    cfg = sp.MgConfig(smoother=M, cycle="V", nu1=1, nu2=1, coarsest_N=2)
    got = host(sp.cycle(sp.Grid(N, dev(x, torch.float32)), sp.Grid(N, dev(b, torch.float32)), cfg))
    ref = c_oracle.cycle(x, b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, 1, 1, 1, 2, dtype=np.float32)
    assert got.dtype == np.float32
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("seed", [1, 2])
def test_random_configs_vs_oracle(seed):
    """Seeded random sweep over the whole cycle path (tests/fuzz_case.py): ragged sizes, every named
    smoother, V / W, nu in 0..2, coarsest_N along the halving chain, fp64 / fp32 and random
    settings of every path switch, two cycles each, bitwise against the C oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "fuzz_case.py"), str(seed), "60"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "FUZZ OK" in r.stdout, (r.stdout[-1500:], r.stderr[-3000:])


def test_random_operators_vs_oracle():
    """Seeded random sweep over the per-operator entry points (tests/fuzz_case.py operators): smooth
    with 0..3 steps at odd and even mesh counts, residual + restriction, prolongation + correction
    and the residual norm, host and device arrays, fp64 and fp32, bitwise against the C oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "fuzz_case.py"), "0", "60", "ops"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "FUZZ OK" in r.stdout, (r.stdout[-1500:], r.stderr[-3000:])


def test_oversized_coarse_system_is_refused():
    """A coarsest level whose unknowns do not fit the single-CTA direct solve is refused with a
    message when the solver is planned (before the LU is even factorised), not with a launch
    failure inside a cycle."""
    from paper_2206_05543_b200._lib import SpaimgError
    cfg = sp.MgConfig(smoother=sp.named("jacobi3d"), cycle="V", nu1=1, nu2=1, coarsest_N=33)
    with pytest.raises(SpaimgError, match="unknowns"):
        sp.Solver(cfg, 3, 66)


def test_long_histories_grow_on_demand():
    """max_iters beyond the initial history capacity (the reference accepts any max_iters,
    multigrid.py:196-201; round 1 capped it at 4096), and more Solver.cycles() than the history
    held: the device history grows, nothing is overwritten, and the start of the history still
    equals the oracle's."""
    N = 16
    b = np.random.default_rng(5).uniform(-1, 1, (N - 1, N - 1))
    M = sp.named("jacobi2d")
    cfg = sp.MgConfig(smoother=M, cycle="V", nu1=1, nu2=0, coarsest_N=2, tol=1e-300, max_iters=5000)
    u, rep = sp.solve(sp.Grid(N, dev(b)), cfg, u0=0)
    assert rep.iterations == 5000 and not rep.converged and len(rep.residual_norms) == 5001
    _, norms, _, _ = c_oracle.solve_history(b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, 1, 0, 1, 2,
                                            tol=1e-300, max_iters=40)
    assert max(abs(a - r) / r for a, r in zip(rep.residual_norms[:41], norms)) < 1e-8
    so = sp.Solver(cfg, 2, N)
    so.load(dev(b))
    so.cycles(300)   # past the 101 norms allocated at creation
    so.cycles(300)
    got = torch.empty((N - 1, N - 1), dtype=torch.float64, device="cuda")
    so.store(got)
    ref = np.zeros_like(b)
    for _ in range(600):
        ref = c_oracle.cycle(ref, b, N, npo.terms_of(M.stencil), M.omega_opt_analytic, 1, 0, 1, 2)
    assert np.array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("seed,shape,dtype", [(0, (4095, 4095), torch.float64), (1, (127, 127, 127), torch.float64),
                                              (12345, (17, 33), torch.float32), (7, (1,), torch.float64)])
def test_device_uniform_is_numpy_bitwise(seed, shape, dtype):
    """The device PCG64 uniform draw equals numpy's default_rng(seed).uniform(0, 1, shape) bit for
    bit (fp32: the float64 draw rounded once)."""
    from paper_2206_05543_b200.multigrid import device_uniform
    like = torch.empty(shape, dtype=dtype, device="cuda")
    got = device_uniform(seed, like).cpu().numpy()
    ref = np.random.default_rng(seed).uniform(0.0, 1.0, shape)
    assert np.array_equal(got, ref.astype(got.dtype))
    got2 = device_uniform(seed, like, -1.0, 1.0).cpu().numpy()
    assert np.array_equal(got2, np.random.default_rng(seed).uniform(-1.0, 1.0, shape).astype(got2.dtype))

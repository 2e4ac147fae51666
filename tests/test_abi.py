"""CPU: the C-ABI library loads and exports every symbol include/spaimg_cuda.h declares;
host-side validation raises the reference's exceptions before any device work."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2206_05543_b200 as sp
from paper_2206_05543_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "spaimg_cuda.h")).read()
    return sorted(set(re.findall(r"SPAIMG_API\s+[\w\s\*]*?\b(spaimg_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("spaimg_smooth", "spaimg_restrict", "spaimg_prolong", "spaimg_cycle", "spaimg_solve",
              "spaimg_apply", "spaimg_residual_norm", "spaimg_solver_create"):
        assert s in syms
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_loads_and_exports_all():
    lib = _lib.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert lib.spaimg_abi_version() == 1
    # no device work: an argument error is reported through the error channel
    rc = lib.spaimg_restrict(0, 2, 7, None, None, None)
    assert rc == -1
    assert b"odd" in lib.spaimg_last_error()


def test_struct_layout_matches_header(tmp_path):
    """ctypes mirrors == the C compiler's layout of the header structs."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    src = tmp_path / "probe.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "spaimg_cuda.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(spaimg_stencil),"
        " sizeof(spaimg_mg_config), offsetof(spaimg_mg_config, omega), offsetof(spaimg_mg_config, coarse_lu),"
        " sizeof(spaimg_solver_stats), offsetof(spaimg_solver_stats, unknowns),"
        " offsetof(spaimg_stencil, coef)); return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    C = _lib
    want = [ctypes.sizeof(C.SpaimgStencil), ctypes.sizeof(C.SpaimgMgConfig), C.SpaimgMgConfig.omega.offset,
            C.SpaimgMgConfig.coarse_lu.offset, ctypes.sizeof(C.SpaimgSolverStats),
            C.SpaimgSolverStats.unknowns.offset, C.SpaimgStencil.coef.offset]
    assert got == want


def test_stencil_marshalling_order():
    from paper_2206_05543_b200.multigrid import _stencil_struct
    st = _stencil_struct(sp.named("m9").stencil)
    assert st.nterms == 9 and st.h_exponent == 2
    offs = [tuple(st.offsets[k][:2]) for k in range(9)]
    assert offs == [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (1, -1), (-1, 1), (-1, -1)]
    assert st.coef[0] == 11 / 6 and st.coef[1] == float(__import__("fractions").Fraction(10, 24))


def test_mgconfig_validation_matches_reference():
    with pytest.raises(ValueError, match="cycle must be"):
        sp.MgConfig(smoother=sp.named("m9"), cycle="X")
    with pytest.raises(ValueError, match="nu1"):
        sp.MgConfig(smoother=sp.named("m9"), nu1=0, nu2=0)
    with pytest.raises(ValueError, match="coarsest_N"):
        sp.MgConfig(smoother=sp.named("m9"), coarsest_N=1)
    with pytest.raises(ValueError, match="tol"):
        sp.MgConfig(smoother=sp.named("m9"), tol=0)
    with pytest.raises(ValueError, match="explicit omega"):
        sp.MgConfig(smoother=sp.upsilon(1, 1, 1)).resolve_smoother()
    with pytest.raises(TypeError, match="NamedSmoother or Stencil"):
        sp.MgConfig(smoother=42).resolve_smoother()
    cfg = sp.MgConfig(smoother=sp.named("m7"))
    assert (cfg.cycle, cfg.nu1, cfg.nu2, cfg.coarsest_N, cfg.tol, cfg.max_iters, cfg.rng_seed) == \
        ("W", 1, 0, 4, 1e-10, 100, 0)


def test_host_validation_before_launch():
    g = sp.Grid(7, np.zeros((6, 6)))
    with pytest.raises(ValueError, match="cannot halve an odd mesh count N=7"):
        sp.restrict(g)
    with pytest.raises(ValueError, match="fine_N must be 2"):
        sp.prolong(sp.Grid(4, np.zeros((3, 3))), 7)
    b = sp.Grid(12, np.zeros((11, 11)))
    with pytest.raises(ValueError, match="must equal coarsest_N"):
        sp.solve(b, sp.MgConfig(smoother=sp.named("m9"), coarsest_N=5))
    with pytest.raises(ValueError, match="smoother dim"):
        sp.solve(sp.Grid(8, np.zeros((7, 7))), sp.MgConfig(smoother=sp.named("m7"), coarsest_N=2))
    with pytest.raises(ValueError, match="same grid"):
        sp.smooth(sp.Grid(8, np.zeros((7, 7))), sp.Grid(4, np.zeros((3, 3))), sp.named("m9").stencil, 0.1, 1)
    with pytest.raises(ValueError, match="does not match interior"):
        sp.Grid(8, np.zeros((6, 6)))


def test_reference_objects_are_accepted_duck_typed():
    class FakeNamed:
        def __init__(self):
            self.stencil = sp.named("m9").stencil
            self.omega_opt_analytic = 0.5
    stencil, om = sp.MgConfig(smoother=FakeNamed()).resolve_smoother()
    assert om == 0.5 and stencil.dim == 2


def test_workload_rhs_matches_golden_hash(golden_hist):
    import hashlib
    from paper_2206_05543_b200 import workloads
    rec = golden_hist["c1/m9/V(1,1)"]
    b = workloads.rhs("c1")
    assert b.shape == (255, 255)
    if hashlib.sha256(b.tobytes()).hexdigest() != rec["sha_b"]:
        pytest.skip("host libm differs from the golden host")

"""Run the reference `spaimg` command line with the GPU hot path dropped in.

This is the integration a reference user makes, not a second CLI: the reference's own
`spaimg.cli` (argument parsing, printout, RunRecord CSV/JSON schema, exit codes, the lfa /
table / verify analysis subcommands) runs unchanged, and its only call into the solver,
`multigrid.solve` (reference cli.py:215-229), is rebound to this package's `solve`, which runs
the cycles on the GPU and hands back the reference's own Grid / SolveReport types.

    python -m paper_2206_05543_b200.cli solve --example 3 --N 64 --cycle v --nu1 1 --nu2 1 --smoother m7
    python -m paper_2206_05543_b200.cli bench --examples 1,3 --Ns 64,128 --cycles v1+1

The reference package must be importable (installed, or its source directory in
SPAIMG_REF_SRC, e.g. /root/reference/pkg/src).  `install()` can also be called from a program
that already imported `spaimg`, to route every later `spaimg.multigrid.solve` / `cycle` call to
the GPU.
"""

import importlib
import os
import sys

__all__ = ["install", "main"]


def _import_reference():
    src = os.environ.get("SPAIMG_REF_SRC")
    if src and src not in sys.path:
        sys.path.insert(0, src)
    try:
        return importlib.import_module("spaimg")
    except ImportError as exc:
        raise SystemExit(f"the reference package `spaimg` is not importable ({exc}); "
                         "install it or set SPAIMG_REF_SRC to its source directory") from exc


def install(spaimg=None):
    """Rebind spaimg.multigrid.solve and .cycle to the GPU implementations (idempotent).
    Returns the reference package."""
    ref = spaimg or _import_reference()
    rmg = importlib.import_module(ref.__name__ + ".multigrid")
    rgrids = importlib.import_module(ref.__name__ + ".grids")
    if getattr(rmg, "_spaimg_b200_installed", False):
        return ref
    from . import multigrid as gmg

    def _host_grid(g):
        return rgrids.Grid(g.N, g.to_host().values)

    def solve(b, cfg):
        u, rep = gmg.solve(b, cfg)
        return _host_grid(u), rmg.SolveReport(iterations=rep.iterations, residual_norms=rep.residual_norms,
                                              rho_hat=rep.rho_hat, converged=rep.converged,
                                              wall_time=rep.wall_time, error_inf=rep.error_inf)

    def cycle(u, b, cfg):
        return _host_grid(gmg.cycle(u, b, cfg))

    rmg._spaimg_b200_cpu = (rmg.solve, rmg.cycle)
    rmg.solve = solve
    rmg.cycle = cycle
    ref.solve = solve
    ref.cycle = cycle
    rmg._spaimg_b200_installed = True
    return ref


def main(argv=None) -> int:
    ref = install()
    cli = importlib.import_module(ref.__name__ + ".cli")
    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())

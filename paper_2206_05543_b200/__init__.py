"""B200-native (sm_100a) geometric-multigrid V/W-cycle with the SPAI smoothers of
arXiv 2206.05543 — a GPU drop-in for the hot path of the reference `spaimg` package.

The exported names are the reference's hot-path API (reference
pkg/src/spaimg/__init__.py:5, :21, :23-33): `Grid`, `Stencil`, `NamedSmoother`,
`laplacian`, `named`, `upsilon`, `tee`, `MgConfig`, `SolveReport`, `smooth`,
`restrict`, `prolong`, `cycle`, `solve`.  Local Fourier analysis, problem
assembly and the CLI stay in the reference (out of scope); `python -m
paper_2206_05543_b200.cli` runs the reference CLI with this package's solve dropped in.
"""

from .grids import Grid
from .multigrid import (MgConfig, SolveReport, Solver, cached_solver, clear_solver_cache, cycle, prolong,
                        prolong_correct, residual_norm, residual_restrict, restrict, smooth, solve)
from .stencils import NAMED_SMOOTHER_IDS, NamedSmoother, Stencil, StencilSymmetryError, laplacian, named, tee, upsilon

__version__ = "0.1.0"

__all__ = [
    "Grid",
    "Stencil",
    "NamedSmoother",
    "StencilSymmetryError",
    "laplacian",
    "named",
    "upsilon",
    "tee",
    "NAMED_SMOOTHER_IDS",
    "MgConfig",
    "SolveReport",
    "smooth",
    "restrict",
    "prolong",
    "cycle",
    "solve",
    "Solver",
    "cached_solver",
    "clear_solver_cache",
    "residual_restrict",
    "prolong_correct",
    "residual_norm",
    "__version__",
]

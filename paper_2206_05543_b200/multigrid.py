"""GPU drop-in for the reference `spaimg.multigrid` API
(reference pkg/src/spaimg/multigrid.py:19-227).

Same names, signatures, defaults, exceptions and return types as the
reference; the work runs in hand-written sm_100a kernels behind the C ABI of
include/spaimg_cuda.h (loaded by `_lib`).  Host (numpy) inputs give host
outputs, CUDA-tensor inputs give CUDA-tensor outputs.  There is no CPU path.

Extensions over the reference (all optional, defaults reproduce it):
  * `solve(b, cfg, u0=None)`: u0=None draws the reference's seeded U(0,1) start
    (multigrid.py:204-205) on the host; pass an array/Grid (or 0) to start elsewhere.
  * float32 device grids (torch float32 tensors) run the fp32 kernels.
  * `solve`/`cycle` keep their device hierarchy and captured graphs between calls
    (`cached_solver`, the counterpart of the reference's lru_cache on the coarse LU).
"""

import ctypes
import threading
import time
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .grids import Grid, is_device_array
from .stencils import NamedSmoother, Stencil, laplacian

__all__ = [
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
]


# ------------------------------------------------------------------------------------------
# configuration and report (multigrid.py:30-83)
# ------------------------------------------------------------------------------------------
def _is_named(sm) -> bool:
    return isinstance(sm, NamedSmoother) or (
        hasattr(sm, "stencil") and hasattr(sm, "omega_opt_analytic"))


def _is_stencil(sm) -> bool:
    return isinstance(sm, Stencil) or (
        hasattr(sm, "entries") and hasattr(sm, "h_exponent") and hasattr(sm, "dim"))


@dataclass
class MgConfig:
    """Multigrid cycle configuration (reference multigrid.py:30-68), same defaults."""

    smoother: object
    cycle: str = "W"
    nu1: int = 1
    nu2: int = 0
    omega: float | None = None
    coarsest_N: int = 4
    tol: float = 1e-10
    max_iters: int = 100
    rng_seed: int = 0

    def __post_init__(self):
        self.cycle = self.cycle.upper()
        if self.cycle not in ("V", "W"):
            raise ValueError(f"cycle must be 'V' or 'W', got {self.cycle!r}")
        if self.nu1 < 0 or self.nu2 < 0 or self.nu1 + self.nu2 < 1:
            raise ValueError("need nu1, nu2 >= 0 with nu1 + nu2 >= 1")
        if self.coarsest_N < 2:
            raise ValueError("coarsest_N must be at least 2")
        if self.tol <= 0:
            raise ValueError("tol must be positive")

    def resolve_smoother(self) -> tuple:
        """(stencil, omega) actually used by the cycles."""
        if _is_named(self.smoother):
            om = self.omega if self.omega is not None else self.smoother.omega_opt_analytic
            return self.smoother.stencil, float(om)
        if _is_stencil(self.smoother):
            if self.omega is None:
                raise ValueError("a custom stencil smoother needs an explicit omega")
            return self.smoother, float(self.omega)
        raise TypeError(f"smoother must be NamedSmoother or Stencil, got {type(self.smoother)}")


@dataclass
class SolveReport:
    """Iteration record of one multigrid solve (reference multigrid.py:71-83)."""

    iterations: int
    residual_norms: list
    rho_hat: float
    converged: bool
    wall_time: float
    error_inf: float | None = None

    def __post_init__(self):
        self.residual_norms = [float(r) for r in self.residual_norms]


# ------------------------------------------------------------------------------------------
# marshalling
# ------------------------------------------------------------------------------------------
def _stencil_struct(S) -> _lib.SpaimgStencil:
    st = _lib.SpaimgStencil()
    items = list(S.entries.items())
    if len(items) > _lib.MAX_TERMS:
        raise ValueError(f"stencil has {len(items)} entries; at most {_lib.MAX_TERMS} are supported")
    st.dim = int(S.dim)
    st.nterms = len(items)
    st.h_exponent = int(S.h_exponent)
    for k, (off, c) in enumerate(items):
        for a in range(3):
            st.offsets[k][a] = int(off[a]) if a < len(off) else 0
        st.coef[k] = float(c)  # reference stencils.py:151
    return st


class _Arr:
    """A grid's values as a raw pointer for the C ABI (keeps the owner alive).

    Device inputs/outputs must be contiguous CUDA tensors of the call's dtype and shape.  Host
    inputs are converted (copied) as needed; host OUTPUTS must already be C-contiguous, writeable
    numpy arrays of the right dtype and shape, since a converted copy would leave the caller's
    array unchanged.
    """

    def __init__(self, values, dtype_code, shape=None, out=False, device=None):
        npdt = np.float64 if dtype_code == _lib.F64 else np.float32
        if is_device_array(values):
            import torch
            want = torch.float64 if dtype_code == _lib.F64 else torch.float32
            if values.dtype != want:
                raise TypeError(f"device array has dtype {values.dtype}, expected {want}")
            if not values.is_contiguous():
                raise ValueError("device array must be contiguous")
            if device is not None and values.device.index != device:
                raise ValueError(f"device array on cuda:{values.device.index}, expected cuda:{device}")
            if shape is not None and tuple(values.shape) != tuple(shape):
                raise ValueError(f"array shape {tuple(values.shape)} does not match {tuple(shape)}")
            self.owner = values
            self.ptr = values.data_ptr()
            return
        try:
            import torch
            if isinstance(values, torch.Tensor):  # CPU tensor: a host array
                values = values.detach().numpy()
        except ImportError:  # pragma: no cover
            pass
        if out:
            if not (isinstance(values, np.ndarray) and values.dtype == npdt and values.flags.c_contiguous
                    and values.flags.writeable):
                raise TypeError(f"host output must be a writeable C-contiguous {np.dtype(npdt).name} numpy array")
            a = values
        else:
            a = np.ascontiguousarray(values, dtype=npdt)
        if shape is not None and tuple(a.shape) != tuple(shape):
            raise ValueError(f"array shape {tuple(a.shape)} does not match {tuple(shape)}")
        self.owner = a
        self.ptr = a.ctypes.data


def _dtype_code(values) -> int:
    if is_device_array(values):
        import torch
        return _lib.F32 if values.dtype == torch.float32 else _lib.F64
    return _lib.F64


def _stream_for(values):
    if is_device_array(values):
        import torch
        _lib.check(_lib.load().spaimg_set_device(values.device.index or 0))
        return ctypes.c_void_p(torch.cuda.current_stream(values.device).cuda_stream)
    _lib.load()
    return ctypes.c_void_p(0)


def _empty_like(values, shape):
    if is_device_array(values):
        import torch
        return torch.empty(shape, dtype=values.dtype, device=values.device)
    return np.empty(shape, dtype=np.float64)


def _same_side(ref, values):
    """Return `values` on the same side (host/device, dtype) as `ref`."""
    if is_device_array(ref):
        import torch
        if is_device_array(values):
            return values.to(device=ref.device, dtype=ref.dtype).contiguous()
        return torch.as_tensor(np.asarray(values, dtype=np.float64)).to(
            device=ref.device, dtype=ref.dtype).contiguous()
    if is_device_array(values):
        return values.detach().cpu().numpy().astype(np.float64)
    return np.ascontiguousarray(values, dtype=np.float64)


# ------------------------------------------------------------------------------------------
# hot-path API
# ------------------------------------------------------------------------------------------
def apply_stencil(S, u: Grid) -> Grid:
    """Stencil.apply on the GPU (reference stencils.py:136-153)."""
    if S.dim != u.dim:
        raise ValueError(f"stencil dim {S.dim} != grid dim {u.dim}")
    lib = _lib.load()
    code = _dtype_code(u.values)
    stream = _stream_for(u.values)
    x = _Arr(u.values, code)
    out = _empty_like(u.values, tuple(u.values.shape))
    o = _Arr(out, code, out=True)
    st = _stencil_struct(S)
    _lib.check(lib.spaimg_apply(code, u.N, ctypes.byref(st), x.ptr, o.ptr, stream))
    return Grid(u.N, out)


def smooth(u: Grid, b: Grid, M, omega: float, steps: int) -> Grid:
    """`steps` damped Richardson sweeps u <- u + omega*M*(b - A*u) (multigrid.py:86-101)."""
    if u.N != b.N or u.dim != b.dim:
        raise ValueError("u and b must live on the same grid")
    if steps < 0:
        raise ValueError("steps must be non-negative")
    if M.dim != u.dim:
        raise ValueError(f"stencil dim {M.dim} != grid dim {u.dim}")
    lib = _lib.load()
    code = _dtype_code(u.values)
    stream = _stream_for(u.values)
    x = _Arr(u.values, code)
    bb = _Arr(_same_side(u.values, b.values), code)
    out = _empty_like(u.values, tuple(u.values.shape))
    o = _Arr(out, code, out=True)
    st = _stencil_struct(M)
    _lib.check(lib.spaimg_smooth(code, u.dim, u.N, x.ptr, bb.ptr, ctypes.byref(st), float(omega), int(steps),
                                 o.ptr, stream))
    return Grid(u.N, out)


def restrict(fine: Grid) -> Grid:
    """Full-weighting restriction to the mesh with half the resolution (multigrid.py:110-119)."""
    if fine.N % 2:
        raise ValueError(f"cannot halve an odd mesh count N={fine.N}")
    if fine.N // 2 < 2:
        raise ValueError("coarse mesh would have no interior points")
    lib = _lib.load()
    code = _dtype_code(fine.values)
    stream = _stream_for(fine.values)
    x = _Arr(fine.values, code)
    Nc = fine.N // 2
    out = _empty_like(fine.values, (Nc - 1,) * fine.dim)
    o = _Arr(out, code, out=True)
    _lib.check(lib.spaimg_restrict(code, fine.dim, fine.N, x.ptr, o.ptr, stream))
    return Grid(Nc, out)


def prolong(coarse: Grid, fine_N: int) -> Grid:
    """d-linear interpolation to the mesh with twice the resolution (multigrid.py:133-144)."""
    if fine_N != 2 * coarse.N:
        raise ValueError(f"fine_N must be 2*{coarse.N}, got {fine_N}")
    lib = _lib.load()
    code = _dtype_code(coarse.values)
    stream = _stream_for(coarse.values)
    e = _Arr(coarse.values, code)
    out = _empty_like(coarse.values, (fine_N - 1,) * coarse.dim)
    o = _Arr(out, code, out=True)
    _lib.check(lib.spaimg_prolong(code, coarse.dim, coarse.N, e.ptr, o.ptr, stream))
    return Grid(fine_N, out)


def residual_restrict(u: Grid, b: Grid) -> Grid:
    """restrict(b - A u) in one fused launch (multigrid.py:176-177)."""
    if u.N != b.N or u.dim != b.dim:
        raise ValueError("u and b must live on the same grid")
    if u.N % 2:
        raise ValueError(f"cannot halve an odd mesh count N={u.N}")
    if u.N // 2 < 2:
        raise ValueError("coarse mesh would have no interior points")
    lib = _lib.load()
    code = _dtype_code(u.values)
    stream = _stream_for(u.values)
    x = _Arr(u.values, code)
    bb = _Arr(_same_side(u.values, b.values), code)
    Nc = u.N // 2
    out = _empty_like(u.values, (Nc - 1,) * u.dim)
    o = _Arr(out, code, out=True)
    _lib.check(lib.spaimg_residual_restrict(code, u.dim, u.N, x.ptr, bb.ptr, o.ptr, stream))
    return Grid(Nc, out)


def prolong_correct(u: Grid, e: Grid) -> Grid:
    """u + prolong(e, u.N) in one fused launch (multigrid.py:184)."""
    if u.N != 2 * e.N or u.dim != e.dim:
        raise ValueError(f"fine_N must be 2*{e.N}, got {u.N}")
    lib = _lib.load()
    code = _dtype_code(u.values)
    stream = _stream_for(u.values)
    x = _Arr(u.values, code)
    ee = _Arr(_same_side(u.values, e.values), code)
    out = _empty_like(u.values, tuple(u.values.shape))
    o = _Arr(out, code, out=True)
    _lib.check(lib.spaimg_prolong_correct(code, u.dim, u.N, x.ptr, ee.ptr, o.ptr, stream))
    return Grid(u.N, out)


def residual_norm(u: Grid, b: Grid) -> float:
    """||b - A u||_2 (multigrid.py:207 / :214)."""
    if u.N != b.N or u.dim != b.dim:
        raise ValueError("u and b must live on the same grid")
    lib = _lib.load()
    code = _dtype_code(u.values)
    stream = _stream_for(u.values)
    x = _Arr(u.values, code)
    bb = _Arr(_same_side(u.values, b.values), code)
    out = ctypes.c_double(0.0)
    _lib.check(lib.spaimg_residual_norm(code, u.dim, u.N, x.ptr, bb.ptr, ctypes.byref(out), stream))
    return float(out.value)


# ------------------------------------------------------------------------------------------
# cycles
# ------------------------------------------------------------------------------------------
_LU_CACHE = {}


def _coarsest_lu(dim: int, N: int):
    """lu_factor of the assembled coarse Laplacian, cached (multigrid.py:147-149).
    Host-side setup: the substitution itself runs on the GPU (K5)."""
    key = (dim, N)
    if key not in _LU_CACHE:
        from scipy.linalg import lu_factor
        lu, piv = lu_factor(laplacian(dim).to_matrix(N).toarray())
        _LU_CACHE[key] = (np.ascontiguousarray(lu, dtype=np.float64),
                          np.ascontiguousarray(piv, dtype=np.int32))
    return _LU_CACHE[key]


def _coarse_level(N: int, coarsest_N: int) -> int:
    """Mesh count at which the recursion solves directly (multigrid.py:166, :178), raising the
    reference's restrict() errors if a halving is impossible on the way (:112-115)."""
    while N > coarsest_N:
        if N % 2:
            raise ValueError(f"cannot halve an odd mesh count N={N}")
        if N // 2 < 2:
            raise ValueError("coarse mesh would have no interior points")
        N //= 2
    return N


def _mg_struct(cfg: MgConfig, dim: int, N: int, dtype_code: int):
    if N <= cfg.coarsest_N:
        # u.N <= coarsest_N: the cycle is the direct solve alone and the reference never looks at
        # the smoother (multigrid.py:166-167); any radius-1 stencil fills the unused slot
        M, omega = laplacian(dim), 0.0
    else:
        M, omega = cfg.resolve_smoother()
        if M.dim != dim:
            raise ValueError(f"smoother dim {M.dim} != grid dim {dim}")
    Nc = _coarse_level(N, cfg.coarsest_N)
    # the device direct solve (K5) keeps the coarse vector in one CTA's shared memory: refuse a
    # larger coarsest level here, before factorising it (the library checks again)
    n_coarse = (Nc - 1) ** dim
    if n_coarse * (8 if dtype_code == _lib.F64 else 4) > 227 * 1024:
        raise _lib.SpaimgError(f"coarsest level N={Nc} has {n_coarse} unknowns, more than the device direct solve "
                               "holds; choose a smaller coarsest_N")
    lu, piv = _coarsest_lu(dim, Nc)
    c = _lib.SpaimgMgConfig()
    c.dtype = dtype_code
    c.dim = dim
    c.N = N
    c.M = _stencil_struct(M)
    c.omega = omega
    c.gamma = 2 if cfg.cycle == "W" else 1
    c.nu1 = int(cfg.nu1)
    c.nu2 = int(cfg.nu2)
    c.coarsest_N = int(cfg.coarsest_N)
    c.coarse_N = Nc
    c.coarse_n = int(lu.shape[0])
    c.coarse_lu = lu.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    c.coarse_piv = piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
    return c, (lu, piv)


# ------------------------------------------------------------------------------------------
# cached solver handles: the reference's only expensive setup is the coarse LU, which it caches
# (lru_cache, multigrid.py:147-149); here the setup is the device hierarchy and the captured
# graphs, cached the same way per (device, dtype, dim, N, smoother terms, omega, cycle shape)
# ------------------------------------------------------------------------------------------
_SOLVER_CACHE = OrderedDict()
_SOLVER_CACHE_MAX = 4
_SOLVER_LOCK = threading.Lock()


def _solver_key(cfg: MgConfig, dim: int, N: int, dtype_code: int, device: int):
    if N <= cfg.coarsest_N:
        sm = None
    else:
        M, omega = cfg.resolve_smoother()
        sm = (int(M.dim), int(M.h_exponent), tuple((tuple(int(v) for v in o), float(c)) for o, c in M.entries.items()),
              float(omega))
    return (device, dtype_code, dim, N, sm, 2 if cfg.cycle == "W" else 1, int(cfg.nu1), int(cfg.nu2),
            int(cfg.coarsest_N))


def cached_solver(cfg: MgConfig, dim: int, N: int, dtype_code: int, device: int = 0) -> "Solver":
    """The Solver for this problem shape, created on first use and kept (LRU, 4 entries); the
    cache holds device memory, clear_solver_cache() releases it."""
    key = _solver_key(cfg, dim, N, dtype_code, device)
    with _SOLVER_LOCK:
        s = _SOLVER_CACHE.get(key)
        if s is not None:
            _SOLVER_CACHE.move_to_end(key)
            return s
    s = Solver(cfg, dim, N, dtype="float32" if dtype_code == _lib.F32 else "float64", device=device)
    with _SOLVER_LOCK:
        _SOLVER_CACHE[key] = s
        while len(_SOLVER_CACHE) > _SOLVER_CACHE_MAX:
            _SOLVER_CACHE.popitem(last=False)
    return s


def clear_solver_cache():
    with _SOLVER_LOCK:
        _SOLVER_CACHE.clear()


def _device_of(values) -> int:
    return (values.device.index or 0) if is_device_array(values) else 0


def cycle(u: Grid, b: Grid, cfg: MgConfig) -> Grid:
    """One multigrid cycle for A*u = b at the grid's resolution (multigrid.py:157-185)."""
    if u.N != b.N or u.dim != b.dim:
        raise ValueError("u and b must live on the same grid")
    _lib.load()
    code = _dtype_code(u.values)
    dev = _device_of(u.values)
    stream = _stream_for(u.values)
    s = cached_solver(cfg, u.dim, u.N, code, dev)
    out = _empty_like(u.values, tuple(u.values.shape))
    with s.lock:
        s.load(_same_side(u.values, b.values), u.values, stream=stream.value)
        s.cycles(1, stream=stream.value)
        s.store(out, stream=stream.value)
    return Grid(u.N, out)


def _check_solve(b: Grid, cfg: MgConfig):
    levels = b.N // cfg.coarsest_N
    if levels * cfg.coarsest_N != b.N or levels & (levels - 1):
        raise ValueError(f"N={b.N} must equal coarsest_N={cfg.coarsest_N} times a power of 2")
    M, _ = cfg.resolve_smoother()
    if M.dim != b.dim:
        raise ValueError(f"smoother dim {M.dim} != problem dim {b.dim}")


def device_uniform(seed, like, low=0.0, high=1.0):
    """np.random.default_rng(seed).uniform(low, high, like.shape) drawn on like's device (bitwise;
    the host only runs numpy's seeding)."""
    import torch
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    out = torch.empty(tuple(like.shape), dtype=like.dtype, device=like.device)
    mask = (1 << 64) - 1
    lib = _lib.load()
    _lib.check(lib.spaimg_fill_uniform(_dtype_code(out), out.numel(), s >> 64, s & mask, inc >> 64, inc & mask,
                                       float(low), float(high), out.data_ptr(), _stream_for(out)))
    return out


def _start_values(b: Grid, cfg: MgConfig, u0):
    """The start iterate: the reference's seeded U(0,1) draw (multigrid.py:204-205) when
    u0 is None; None (zero start, no upload) when u0 is 0; else the given values."""
    if u0 is None:
        if is_device_array(b.values):  # drawn on the device, bitwise the numpy draw
            return device_uniform(cfg.rng_seed, b.values, 0.0, 1.0)
        rng = np.random.default_rng(cfg.rng_seed)
        return _same_side(b.values, rng.uniform(0.0, 1.0, size=tuple(b.values.shape)))
    if isinstance(u0, (int, float)) and u0 == 0:
        return None
    vals = u0.values if hasattr(u0, "values") else u0
    if tuple(vals.shape) != tuple(b.values.shape):
        raise ValueError("u0 must have the shape of b")
    return _same_side(b.values, vals)


def solve(b: Grid, cfg: MgConfig, u0=None) -> tuple:
    """Run cycles from the start until ||r_k|| <= tol ||r_0|| or max_iters (multigrid.py:188-227).

    Returns (solution Grid, SolveReport); rho_hat = (||r_K|| / ||r_0||)**(1/K).  The device
    hierarchy and graphs are cached across calls (cached_solver).
    """
    _check_solve(b, cfg)
    _lib.load()
    code = _dtype_code(b.values)
    dev = _device_of(b.values)
    stream = _stream_for(b.values)
    t0 = time.perf_counter()
    s = cached_solver(cfg, b.dim, b.N, code, dev)
    start = _start_values(b, cfg, u0)
    out = _empty_like(b.values, tuple(b.values.shape))
    with s.lock:
        s.load(b.values, start, stream=stream.value)
        hist, k, conv = s.run(cfg.tol, cfg.max_iters, stream=stream.value)
        s.store(out, stream=stream.value)
    rho_hat = (hist[-1] / hist[0]) ** (1.0 / k) if k else float("nan")
    report = SolveReport(iterations=k, residual_norms=hist, rho_hat=float(rho_hat), converged=conv,
                         wall_time=time.perf_counter() - t0)
    return Grid(b.N, out), report


# ------------------------------------------------------------------------------------------
# persistent solver handle (cached by solve/cycle; also the bench / batch API)
# ------------------------------------------------------------------------------------------
class Solver:
    """Owns the device level hierarchy and the captured cycle graph for one (cfg, N, dtype)."""

    def __init__(self, cfg: MgConfig, dim: int, N: int, dtype: str = "float64", device=0):
        self.cfg = cfg
        self.dim = dim
        self.N = N
        self.device = int(device)
        self.dtype_code = _lib.F32 if dtype in ("float32", "f32", "fp32") else _lib.F64
        self.shape = (N - 1,) * dim
        self.lock = threading.Lock()
        self.lib = _lib.load()
        _lib.check(self.lib.spaimg_set_device(self.device))
        c, self._keep = _mg_struct(cfg, dim, N, self.dtype_code)
        self._cfg_struct = c
        h = ctypes.c_void_p()
        _lib.check(self.lib.spaimg_solver_create(ctypes.byref(c), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.lib.spaimg_solver_destroy(h)
            self.handle = None

    def _stream(self, stream):
        if stream is None:
            import torch
            return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        return ctypes.c_void_p(stream)

    def _ptr(self, values, out=False):
        """Validated pointer to an (N-1)^dim array of the solver's dtype on its device or the host."""
        if values is None:
            return None, None
        a = _Arr(values, self.dtype_code, shape=self.shape, out=out, device=self.device)
        return a, a.ptr

    def load(self, b_values, u0_values=None, stream=None):
        bk, bp = self._ptr(b_values)
        uk, up = self._ptr(u0_values)
        _lib.check(self.lib.spaimg_solver_load(self.handle, bp, up, self._stream(stream)))

    def cycles(self, n, stream=None):
        _lib.check(self.lib.spaimg_solver_cycles(self.handle, int(n), self._stream(stream)))

    def run(self, tol=None, max_iters=None, stream=None):
        tol = self.cfg.tol if tol is None else tol
        max_iters = self.cfg.max_iters if max_iters is None else max_iters
        norms = (ctypes.c_double * (max_iters + 1))()
        iters = ctypes.c_int(0)
        conv = ctypes.c_int(0)
        _lib.check(self.lib.spaimg_solver_run(self.handle, float(tol), int(max_iters), norms, ctypes.byref(iters),
                                              ctypes.byref(conv), self._stream(stream)))
        k = iters.value
        return [float(norms[i]) for i in range(k + 1)], k, bool(conv.value)

    def solve_batch(self, b_list, u_list, tol=None, max_iters=None, stream=None):
        """Independent zero-start solves of each b in `b_list` into the matching `u_list` array,
        pipelined so that host<->device copies overlap the solves (pass pinned host arrays or
        device tensors).  Returns [(residual_norms, iterations, converged), ...]."""
        if len(b_list) != len(u_list):
            raise ValueError("b_list and u_list must have the same length")
        tol = self.cfg.tol if tol is None else tol
        max_iters = self.cfg.max_iters if max_iters is None else max_iters
        n = len(b_list)
        keep = [self._ptr(v)[0] for v in b_list] + [self._ptr(v, out=True)[0] for v in u_list]
        bp = (ctypes.c_void_p * n)(*[k.ptr for k in keep[:n]])
        up = (ctypes.c_void_p * n)(*[k.ptr for k in keep[n:]])
        norms = (ctypes.c_double * (n * (max_iters + 1)))()
        iters = (ctypes.c_int * n)()
        conv = (ctypes.c_int * n)()
        _lib.check(self.lib.spaimg_solver_solve_batch(self.handle, n, bp, up, float(tol), int(max_iters), norms, iters,
                                                      conv, self._stream(stream)))
        out = []
        for i in range(n):
            k = iters[i]
            out.append(([float(norms[i * (max_iters + 1) + j]) for j in range(k + 1)], k, bool(conv[i])))
        del keep
        return out

    def store(self, out_values, stream=None):
        ok, op = self._ptr(out_values, out=True)
        _lib.check(self.lib.spaimg_solver_store(self.handle, op, self._stream(stream)))

    def op(self, which, reps=1, stream=None):
        _lib.check(self.lib.spaimg_solver_op(self.handle, int(which), int(reps), self._stream(stream)))

    def stats(self) -> dict:
        st = _lib.SpaimgSolverStats()
        _lib.check(self.lib.spaimg_solver_stats_get(self.handle, ctypes.byref(st)))
        return {f: getattr(st, f) for f, _ in st._fields_}

"""ctypes binding of libspaimg_cuda.so (the C ABI in include/spaimg_cuda.h).

There is no CPU fallback: if the library cannot be loaded, importing the
hot-path functions raises.
"""

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# SPAIMG_DEBUG=1 selects the checked build (NaN poisoning + barrier jitter; build.py --debug)
DEBUG = os.environ.get("SPAIMG_DEBUG") == "1"
LIB_PATH = os.path.join(_PKG, "libspaimg_cuda_debug.so" if DEBUG else "libspaimg_cuda.so")
# test hook: load another build of the same ABI (the checked-build self-test's fault injection)
LIB_PATH = os.environ.get("SPAIMG_LIB_OVERRIDE") or LIB_PATH

F64 = 0
F32 = 1
MAX_TERMS = 27


class SpaimgStencil(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int),
        ("nterms", ctypes.c_int),
        ("h_exponent", ctypes.c_int),
        ("offsets", (ctypes.c_int * 3) * MAX_TERMS),
        ("coef", ctypes.c_double * MAX_TERMS),
    ]


class SpaimgMgConfig(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int),
        ("dim", ctypes.c_int),
        ("N", ctypes.c_int),
        ("M", SpaimgStencil),
        ("omega", ctypes.c_double),
        ("gamma", ctypes.c_int),
        ("nu1", ctypes.c_int),
        ("nu2", ctypes.c_int),
        ("coarsest_N", ctypes.c_int),
        ("coarse_N", ctypes.c_int),
        ("coarse_n", ctypes.c_int),
        ("coarse_lu", ctypes.POINTER(ctypes.c_double)),
        ("coarse_piv", ctypes.POINTER(ctypes.c_int)),
    ]


class SpaimgSolverStats(ctypes.Structure):
    _fields_ = [
        ("levels", ctypes.c_int),
        ("kernels_per_cycle", ctypes.c_int),
        ("bytes_per_cycle", ctypes.c_double),
        ("unknowns", ctypes.c_longlong),
        ("graph", ctypes.c_int),
        ("fused_sweep", ctypes.c_int),
        ("kernels_stop_test", ctypes.c_int),
    ]


# every exported symbol, with its argtypes (None = leave default)
_VP = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_PD = ctypes.POINTER(ctypes.c_double)
_PI = ctypes.POINTER(ctypes.c_int)
_PS = ctypes.POINTER(SpaimgStencil)
_PC = ctypes.POINTER(SpaimgMgConfig)

SIGNATURES = {
    "spaimg_last_error": ([], ctypes.c_char_p),
    "spaimg_abi_version": ([], _I),
    "spaimg_set_device": ([_I], _I),
    "spaimg_apply": ([_I, _I, _PS, _VP, _VP, _VP], _I),
    "spaimg_smooth": ([_I, _I, _I, _VP, _VP, _PS, _D, _I, _VP, _VP], _I),
    "spaimg_restrict": ([_I, _I, _I, _VP, _VP, _VP], _I),
    "spaimg_prolong": ([_I, _I, _I, _VP, _VP, _VP], _I),
    "spaimg_residual_restrict": ([_I, _I, _I, _VP, _VP, _VP, _VP], _I),
    "spaimg_prolong_correct": ([_I, _I, _I, _VP, _VP, _VP, _VP], _I),
    "spaimg_residual_norm": ([_I, _I, _I, _VP, _VP, _PD, _VP], _I),
    "spaimg_cycle": ([_PC, _VP, _VP, _VP, _VP], _I),
    "spaimg_solve": ([_PC, _VP, _VP, _VP, _D, _I, _PD, _PI, _PI, _VP], _I),
    "spaimg_solver_create": ([_PC, ctypes.POINTER(_VP)], _I),
    "spaimg_solver_destroy": ([_VP], _I),
    "spaimg_solver_stats_get": ([_VP, ctypes.POINTER(SpaimgSolverStats)], _I),
    "spaimg_solver_load": ([_VP, _VP, _VP, _VP], _I),
    "spaimg_solver_cycles": ([_VP, _I, _VP], _I),
    "spaimg_solver_run": ([_VP, _D, _I, _PD, _PI, _PI, _VP], _I),
    "spaimg_solver_store": ([_VP, _VP, _VP], _I),
    "spaimg_fill_uniform": ([_I, ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_ulonglong,
                             ctypes.c_ulonglong, _D, _D, _VP, _VP], _I),
    "spaimg_solver_solve_batch": ([_VP, _I, ctypes.POINTER(_VP), ctypes.POINTER(_VP), _D, _I, _PD, _PI, _PI, _VP], _I),
    "spaimg_solver_op": ([_VP, _I, _I, _VP], _I),
}

_lib = None


class SpaimgError(RuntimeError):
    pass


def load():
    """Load (building in-tree first if needed) the CUDA library; raise if impossible."""
    global _lib
    if _lib is not None:
        return _lib
    from . import build as _build
    try:
        if os.environ.get("SPAIMG_LIB_OVERRIDE"):
            raise RuntimeError("prebuilt library requested")
        _build.build(force=os.environ.get("SPAIMG_REBUILD") == "1", debug=DEBUG)  # no-op when up to date
    except Exception as exc:  # no nvcc / failed build: a prebuilt library is still acceptable
        if not os.path.exists(LIB_PATH):
            raise SpaimgError(f"cannot build the spaimg CUDA library: {exc}") from exc
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise SpaimgError(f"cannot load the spaimg CUDA library {LIB_PATH}: {exc}") from exc
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.spaimg_abi_version() != 1:
        raise SpaimgError("spaimg CUDA library ABI mismatch")
    _lib = lib
    return lib


def check(rc):
    if rc != 0:
        msg = _lib.spaimg_last_error().decode(errors="replace") if _lib is not None else "?"
        raise SpaimgError(f"spaimg CUDA call failed ({rc}): {msg}")

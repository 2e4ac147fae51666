"""ctypes wrapper over the C oracle (`oracle/spaimg_oracle.c`) — TEST INFRASTRUCTURE ONLY.

Same semantics as `oracle.numpy_oracle`, fp64 and fp32, with OpenMP threads;
used as the checker at full sizes and as the timed CPU baseline in bench.py.
"""

import ctypes
import os
import subprocess

import numpy as np

from . import numpy_oracle as npo

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build(force=False):
    so = os.path.join(_HERE, "liboracle.so")
    if force or not os.path.exists(so):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return so


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build())
        for sfx in ("_f64", "_f32"):
            getattr(_LIB, "oracle_residual_norm" + sfx).restype = ctypes.c_double
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _sfx(dtype):
    dt = np.dtype(dtype)
    if dt == np.float64:
        return "_f64", ctypes.c_double, np.float64
    if dt == np.float32:
        return "_f32", ctypes.c_float, np.float32
    raise ValueError(f"unsupported dtype {dt}")


def _terms(terms, dim, dt):
    offs = np.ascontiguousarray([o for off, _ in terms for o in off], dtype=np.int32)
    assert offs.size == dim * len(terms)
    coef = np.ascontiguousarray([c for _, c in terms], dtype=dt)
    return len(terms), offs, coef


def max_threads():
    return int(lib().oracle_max_threads())


def set_threads(n):
    lib().oracle_set_threads(int(n))


def _scale(N, e, dt):
    return dt((1.0 / N) ** e)


def smooth(x, b, N, mterms, omega, steps, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    x = np.ascontiguousarray(x, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    out = np.empty_like(x)
    nt, offs, coef = _terms(mterms, x.ndim, dt)
    rc = getattr(lib(), "oracle_smooth" + sfx)(
        x.ndim, N, _p(x), _p(b), _p(out), nt, _p(offs), _p(coef),
        cty(_scale(N, -2, dt)), cty(_scale(N, 2, dt)), cty(dt(omega)), int(steps))
    assert rc == 0
    return out


def apply(x, N, terms, h_exp, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    x = np.ascontiguousarray(x, dtype=dt)
    out = np.empty_like(x)
    nt, offs, coef = _terms(terms, x.ndim, dt)
    getattr(lib(), "oracle_apply" + sfx)(x.ndim, N, _p(x), _p(out), nt, _p(offs), _p(coef),
                                         cty(_scale(N, h_exp, dt)))
    return out


def residual_restrict(x, b, N, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    x = np.ascontiguousarray(x, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    out = np.empty((N // 2 - 1,) * x.ndim, dtype=dt)
    rc = getattr(lib(), "oracle_residual_restrict" + sfx)(x.ndim, N, _p(x), _p(b), _p(out),
                                                          cty(_scale(N, -2, dt)))
    assert rc == 0
    return out


def prolong_correct(x, e, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    out = np.array(x, dtype=dt, copy=True, order="C")
    e = np.ascontiguousarray(e, dtype=dt)
    Nc = e.shape[0] + 1
    rc = getattr(lib(), "oracle_prolong_correct" + sfx)(e.ndim, Nc, _p(out), _p(e))
    assert rc == 0
    return out


def residual_norm(x, b, N, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    x = np.ascontiguousarray(x, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    return float(getattr(lib(), "oracle_residual_norm" + sfx)(x.ndim, N, _p(x), _p(b)))


def lu_solve(lu, piv, b, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    lu = np.ascontiguousarray(lu, dtype=dt)
    piv = np.ascontiguousarray(piv, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=dt).ravel()
    x = np.empty_like(b)
    getattr(lib(), "oracle_lu_solve" + sfx)(int(b.size), _p(lu), _p(piv), _p(b), _p(x))
    return x


def _coarse(dim, coarsest_N, dt):
    lu, piv = npo.coarse_lu(dim, coarsest_N)
    return (np.ascontiguousarray(lu, dtype=dt), np.ascontiguousarray(piv, dtype=np.int32))


def cycle(x, b, N, mterms, omega, nu1, nu2, gamma, coarsest_N, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    u = np.array(x, dtype=dt, copy=True, order="C")
    b = np.ascontiguousarray(b, dtype=dt)
    nt, offs, coef = _terms(mterms, u.ndim, dt)
    lu, piv = _coarse(u.ndim, min(N, coarsest_N) if N <= coarsest_N else _coarsest_level(N, coarsest_N), dt)
    rc = getattr(lib(), "oracle_cycle" + sfx)(
        u.ndim, N, _p(u), _p(b), nt, _p(offs), _p(coef), cty(dt(omega)), nu1, nu2, gamma,
        coarsest_N, lu.shape[0], _p(lu), _p(piv))
    assert rc == 0
    return u


def _coarsest_level(N, coarsest_N):
    """Mesh count where the recursion stops (first N <= coarsest_N when halving)."""
    while N > coarsest_N:
        N //= 2
    return N


def solve_history(b, N, mterms, omega, nu1=1, nu2=1, gamma=1, coarsest_N=2, tol=1e-10,
                  max_iters=100, u0=None, dtype=np.float64):
    sfx, cty, dt = _sfx(dtype)
    b = np.ascontiguousarray(b, dtype=dt)
    u = np.zeros_like(b) if u0 is None else np.array(u0, dtype=dt, copy=True, order="C")
    nt, offs, coef = _terms(mterms, u.ndim, dt)
    lu, piv = _coarse(u.ndim, _coarsest_level(N, coarsest_N), dt)
    norms = np.zeros(max_iters + 1)
    iters = ctypes.c_int(0)
    conv = ctypes.c_int(0)
    rc = getattr(lib(), "oracle_solve" + sfx)(
        u.ndim, N, _p(u), _p(b), nt, _p(offs), _p(coef), cty(dt(omega)), nu1, nu2, gamma,
        coarsest_N, lu.shape[0], _p(lu), _p(piv), ctypes.c_double(tol), max_iters, _p(norms),
        ctypes.byref(iters), ctypes.byref(conv))
    assert rc == 0
    k = iters.value
    return u, [float(v) for v in norms[: k + 1]], k, bool(conv.value)

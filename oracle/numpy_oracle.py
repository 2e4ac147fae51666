"""numpy restatement of the spaimg V-cycle hot path — TEST INFRASTRUCTURE ONLY.

Every function restates one reference function with the exact per-point
expression tree of SURVEY.md Appendix A, in float64 (bitwise equal to the
reference) and in float32 (the build-defined fp32 contract, Appendix A.8:
constants rounded once to float32, every operation a single float32 rounding).

Inputs are plain C-ordered ndarrays of interior values (reference
`grids.py:10-56`); stencils are given as ordered term lists
`[(offset_tuple, float(coef)), ...]` in `entries` insertion order
(reference `stencils.py:149-151`).
"""

import numpy as np
from scipy.linalg import lu_factor, lu_solve

__all__ = [
    "terms_of", "laplacian_terms", "apply", "residual", "smooth", "restrict",
    "prolong", "prolong_correct", "residual_restrict", "coarse_lu", "coarse_solve",
    "cycle", "residual_norm", "solve_history",
]


def _dt(dtype):
    dt = np.dtype(dtype)
    if dt not in (np.float64, np.float32):
        raise ValueError(f"unsupported dtype {dt}")
    return dt.type


def terms_of(stencil):
    """Ordered (offset, float(c)) list — reference stencils.py:149-151."""
    return [(tuple(int(v) for v in o), float(c)) for o, c in stencil.entries.items()]


def laplacian_terms(dim):
    """reference stencils.py:209-223 (centre, then +-axis0, +-axis1[, +-axis2])."""
    if dim == 2:
        t = [((0, 0), 4.0)]
        t += [(o, -1.0) for o in ((1, 0), (-1, 0), (0, 1), (0, -1))]
        return t
    if dim == 3:
        t = [((0, 0, 0), 6.0)]
        for axis in range(3):
            for s in (1, -1):
                t.append((tuple(s if a == axis else 0 for a in range(3)), -1.0))
        return t
    raise ValueError(f"dim must be 2 or 3, got {dim}")


def _scale(N, h_exp, dt):
    # reference stencils.py:152 — `u.h ** self.h_exponent` with u.h = 1.0 / N (grids.py:38-40)
    return dt((1.0 / N) ** h_exp)


def apply(x, N, terms, h_exp, dtype=np.float64):
    """Zero-extended stencil product — reference stencils.py:136-153."""
    dt = _dt(dtype)
    x = np.asarray(x, dtype=dt)
    w = max(max(abs(o) for o in off) for off, _ in terms)
    padded = np.pad(x, w) if w else x
    out = np.zeros_like(x)
    for off, c in terms:
        sl = tuple(slice(w + o, w + o + n) for o, n in zip(off, x.shape))
        out += dt(c) * padded[sl]
    out *= _scale(N, h_exp, dt)
    return out


def residual(x, b, N, dtype=np.float64):
    """r = b - A x — reference multigrid.py:99 / :176 / :207."""
    dt = _dt(dtype)
    x = np.asarray(x, dtype=dt)
    return np.asarray(b, dtype=dt) - apply(x, N, laplacian_terms(x.ndim), -2, dt)


def smooth(x, b, N, mterms, omega, steps, m_hexp=2, dtype=np.float64):
    """`steps` sweeps v <- v + omega*(M(b - A v)) — reference multigrid.py:86-101."""
    dt = _dt(dtype)
    v = np.array(x, dtype=dt, copy=True)
    om = dt(omega)
    for _ in range(steps):
        r = residual(v, b, N, dt)
        v += om * apply(r, N, mterms, m_hexp, dt)
    return v


def _restrict_axis(a, axis):
    a = np.moveaxis(a, axis, 0)
    out = 0.25 * a[0:-2:2] + 0.5 * a[1:-1:2] + 0.25 * a[2::2]
    return np.moveaxis(out, 0, axis)


def restrict(r):
    """Full weighting, axis 0 first — reference multigrid.py:104-119."""
    v = np.asarray(r)
    if (v.shape[0] + 1) % 2 or (v.shape[0] + 1) // 2 < 2:
        raise ValueError("restrict needs an even mesh count with N/2 >= 2")
    for axis in range(v.ndim):
        v = _restrict_axis(v, axis)
    return v


def _prolong_axis(a, axis):
    a = np.moveaxis(a, axis, 0)
    m = a.shape[0]
    out = np.zeros((2 * m + 1,) + a.shape[1:], dtype=a.dtype)
    out[1::2] = a
    out[2:-2:2] = 0.5 * (a[:-1] + a[1:])
    out[0] = 0.5 * a[0]
    out[-1] = 0.5 * a[-1]
    return np.moveaxis(out, 0, axis)


def prolong(e):
    """d-linear interpolation, axis 0 first — reference multigrid.py:122-144."""
    v = np.asarray(e)
    for axis in range(v.ndim):
        v = _prolong_axis(v, axis)
    return v


def prolong_correct(x, e):
    """v + prolong(ec) — reference multigrid.py:184."""
    return np.asarray(x) + prolong(np.asarray(e, dtype=np.asarray(x).dtype))


def residual_restrict(x, b, N, dtype=np.float64):
    """restrict(b - A v) — reference multigrid.py:176-177."""
    return restrict(residual(x, b, N, dtype))


_LU_CACHE = {}


def coarse_lu(dim, N):
    """lu_factor of the assembled Laplacian — reference multigrid.py:147-149,
    matrix of stencils.py:155-174 (entries float(c) * (1.0/N)**-2)."""
    key = (dim, N)
    if key not in _LU_CACHE:
        n = N - 1
        shape = (n,) * dim
        size = n ** dim
        scale = (1.0 / N) ** -2
        A = np.zeros((size, size))
        idx = np.indices(shape).reshape(dim, -1)
        for off, c in laplacian_terms(dim):
            j = idx + np.asarray(off)[:, None]
            ok = np.all((j >= 0) & (j < n), axis=0)
            rows = np.ravel_multi_index(tuple(idx[:, ok]), shape)
            cols = np.ravel_multi_index(tuple(j[:, ok]), shape)
            A[rows, cols] += float(c) * scale
        _LU_CACHE[key] = lu_factor(A)
    return _LU_CACHE[key]


def coarse_solve(b, N, dtype=np.float64):
    """Direct coarsest solve — reference multigrid.py:152-154.

    float64: scipy lu_solve, exactly the reference call.  float32 (build
    contract): only the 1x1 case N=2 is restated here, x = b / float32(a)
    (Appendix A.5); larger fp32 coarse solves are restated in C (fmaf order).
    """
    dt = _dt(dtype)
    b = np.asarray(b, dtype=dt)
    dim = b.ndim
    if dt is np.float64:
        return lu_solve(coarse_lu(dim, N), b.ravel()).reshape(b.shape)
    if N != 2:
        raise NotImplementedError("fp32 coarse solve for N>2 lives in the C oracle")
    a = dt(float(2 * dim) * ((1.0 / N) ** -2))
    return b / a


def cycle(x, b, N, mterms, omega, nu1, nu2, gamma, coarsest_N, m_hexp=2, dtype=np.float64):
    """One V (gamma=1) / W (gamma=2) cycle — reference multigrid.py:157-185."""
    dt = _dt(dtype)
    if N <= coarsest_N:
        return coarse_solve(b, N, dt)
    v = smooth(x, b, N, mterms, omega, nu1, m_hexp, dt)
    rc = residual_restrict(v, b, N, dt)
    Nc = N // 2
    if Nc <= coarsest_N:
        ec = coarse_solve(rc, Nc, dt)
    else:
        ec = np.zeros_like(rc)
        for _ in range(gamma):
            ec = cycle(ec, rc, Nc, mterms, omega, nu1, nu2, gamma, coarsest_N, m_hexp, dt)
    v = prolong_correct(v, ec)
    return smooth(v, b, N, mterms, omega, nu2, m_hexp, dt)


def residual_norm(x, b, N, dtype=np.float64):
    """||b - A u||_2 — reference multigrid.py:207/214 (reduction order free, A.7)."""
    r = residual(x, b, N, dtype).astype(np.float64)
    return float(np.linalg.norm(r.ravel()))


def solve_history(b, N, mterms, omega, nu1=1, nu2=1, gamma=1, coarsest_N=2,
                  tol=1e-10, max_iters=100, u0=None, dtype=np.float64):
    """solve() loop (reference multigrid.py:206-219) from a given start
    (default zero).  Returns (u, norms, iterations, converged)."""
    dt = _dt(dtype)
    b = np.asarray(b, dtype=dt)
    u = np.zeros_like(b) if u0 is None else np.array(u0, dtype=dt)
    norms = [residual_norm(u, b, N, dt)]
    k = 0
    converged = False
    while k < max_iters:
        u = cycle(u, b, N, mterms, omega, nu1, nu2, gamma, coarsest_N, dtype=dt)
        k += 1
        norms.append(residual_norm(u, b, N, dt))
        if norms[-1] <= tol * norms[0]:
            converged = True
            break
    return u, norms, k, converged

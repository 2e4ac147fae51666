"""Seeded synthetic inputs of the BASELINE.json configs (lines 7-11).

The reference has no benchmark suite: configs 1 and 3 are manufactured sine
problems assembled like reference `problems.assemble_rhs` (problems.py:64-90,
g = None), configs 2, 4 and 5 draw i.i.d. U[-1, 1] right-hand sides with numpy's
default_rng.  Inputs are generated once on the host and the same arrays feed the
GPU path and the CPU baseline.
"""

import math

import numpy as np

__all__ = ["CONFIGS", "rhs", "microbench_inputs"]

CONFIGS = {
    # id: (dim, N, description)
    "c1": (2, 256, "2D sine, h=1/256, m9 V(1,1), zero start, coarsest h=1/2"),
    "c2": (2, 4096, "2D U[-1,1] seed 0, h=1/4096, m9/jacobi2d V(1,1)/V(2,2), zero start"),
    "c3": (3, 128, "3D sine, h=1/128, m7 V(1,1), zero start"),
    "c4": (3, 512, "3D U[-1,1] seed 1, h=1/512, m7/jacobi3d V(1,1)/V(2,2), zero start"),
}


def _mesh(dim, N):
    x = np.arange(1, N) * (1.0 / N)
    return np.meshgrid(*([x] * dim), indexing="ij")


def rhs(cfg_id: str) -> np.ndarray:
    """Right-hand side of config `cfg_id` as a float64 C-ordered array of (N-1)^dim values."""
    if cfg_id == "c1":
        X, Y = _mesh(2, 256)
        return np.ascontiguousarray(2 * math.pi ** 2 * np.sin(math.pi * X) * np.sin(math.pi * Y), dtype=float)
    if cfg_id == "c3":
        X, Y, Z = _mesh(3, 128)
        return np.ascontiguousarray(3 * math.pi ** 2 * np.sin(math.pi * X) * np.sin(math.pi * Y)
                                    * np.sin(math.pi * Z), dtype=float)
    if cfg_id == "c2":
        return np.random.default_rng(0).uniform(-1, 1, (4095, 4095))
    if cfg_id == "c4":
        return np.random.default_rng(1).uniform(-1, 1, (511, 511, 511))
    raise KeyError(cfg_id)


def microbench_inputs(dim: int, N: int, dtype=np.float64):
    """Config 5: x then b then the coarse e, all U[-1,1] from seed 2."""
    rng = np.random.default_rng(2)
    shape = (N - 1,) * dim
    x = rng.uniform(-1, 1, shape)
    b = rng.uniform(-1, 1, shape)
    e = rng.uniform(-1, 1, (N // 2 - 1,) * dim)
    return x.astype(dtype), b.astype(dtype), e.astype(dtype)

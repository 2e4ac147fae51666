"""Grid of interior unknowns — mirror of the reference `spaimg.grids.Grid`
(reference pkg/src/spaimg/grids.py:10-56).

`values` is either a host numpy array (coerced to float64 exactly like the
reference, grids.py:24) or a CUDA `torch.Tensor` of dtype float64 or float32
(device-resident grids; float32 is the build's extra precision, SURVEY.md
Appendix A.8).  Hot-path functions return grids on the same side as their
inputs: host in -> host out, device in -> device out.
"""

from dataclasses import dataclass

import numpy as np

__all__ = ["Grid", "is_device_array"]


def is_device_array(v) -> bool:
    """True for CUDA tensors only; CPU torch tensors count as host arrays."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, torch.Tensor) and v.is_cuda


@dataclass
class Grid:
    """Interior values of a function on a uniform mesh of [0,1]^dim (h = 1/N)."""

    N: int
    values: object

    def __post_init__(self):
        if is_device_array(self.values):
            import torch
            v = self.values
            if v.dtype not in (torch.float64, torch.float32):
                v = v.to(torch.float64)
            self.values = v.contiguous()
            shape = tuple(self.values.shape)
            ndim = self.values.dim()
        else:
            self.values = np.asarray(self.values, dtype=float)
            shape = self.values.shape
            ndim = self.values.ndim
        if self.N < 2:
            raise ValueError(f"need N >= 2, got N={self.N}")
        expected = (self.N - 1,) * ndim
        if shape != expected:
            raise ValueError(
                f"values shape {shape} does not match interior "
                f"of an N={self.N} mesh (expected {expected})"
            )

    @property
    def dim(self) -> int:
        return len(self.values.shape)

    @property
    def h(self) -> float:
        return 1.0 / self.N

    @property
    def on_device(self) -> bool:
        return is_device_array(self.values)

    @classmethod
    def zeros(cls, dim: int, N: int, device=None, dtype=None) -> "Grid":
        if device is None:
            return cls(N, np.zeros((N - 1,) * dim))
        import torch
        return cls(N, torch.zeros((N - 1,) * dim, dtype=dtype or torch.float64, device=device))

    def copy(self) -> "Grid":
        return Grid(self.N, self.values.clone() if self.on_device else self.values.copy())

    def norm2(self) -> float:
        """Euclidean norm of the interior values."""
        if self.on_device:
            import torch
            return float(torch.linalg.vector_norm(self.values.reshape(-1).double()))
        return float(np.linalg.norm(self.values.ravel()))

    def interior_coordinates(self):
        """Tuple of dim arrays (meshgrid, ij indexing) of interior point coordinates."""
        x = np.arange(1, self.N) * self.h
        return np.meshgrid(*([x] * self.dim), indexing="ij")

    def to_host(self) -> "Grid":
        if self.on_device:
            return Grid(self.N, self.values.cpu().numpy().astype(np.float64, copy=False))
        return self

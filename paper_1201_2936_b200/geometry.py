"""Host-side containers mirroring the reference's ``PointSet`` and
``Tolerance`` (/root/reference/pkg/src/seghull/geometry.py:24-83).

Only the containers live here; all predicates run on the device
(csrc/sh_numerics.cuh).  ``Tolerance.effective`` is computed on the device
as well (eps_rel * glibc-hypot of the bbox spans, K0 in csrc/sh_kernels.cuh).
"""

from dataclasses import dataclass

import numpy as np

from .errors import ContractViolation

DEFAULT_EPS_REL = 1e-12


@dataclass(frozen=True)
class PointSet:
    """Structure-of-arrays point collection, 2D or 3D, float64
    (geometry.py:24-65)."""

    coords: tuple

    def __post_init__(self):
        arrays = tuple(np.ascontiguousarray(c, dtype=np.float64) for c in self.coords)
        object.__setattr__(self, "coords", arrays)
        if len(arrays) not in (2, 3):
            raise ContractViolation(f"points must be 2D or 3D, got {len(arrays)} axes")
        n = arrays[0].size
        for c in arrays:
            if c.ndim != 1 or c.size != n:
                raise ContractViolation("coordinate arrays must be 1D and equal length")
            if c.size and not np.isfinite(c).all():
                raise ContractViolation("coordinates must be finite")

    @property
    def dim(self) -> int:
        return len(self.coords)

    @property
    def n(self) -> int:
        return self.coords[0].size

    @classmethod
    def from_rows(cls, rows) -> "PointSet":
        m = np.atleast_2d(np.asarray(rows, dtype=np.float64))
        if m.size == 0:
            raise ContractViolation("from_rows needs an (n, dim) array; use empty() for n=0")
        return cls(tuple(m[:, j].copy() for j in range(m.shape[1])))

    @classmethod
    def empty(cls, dim: int) -> "PointSet":
        return cls(tuple(np.empty(0, np.float64) for _ in range(dim)))

    def as_rows(self) -> np.ndarray:
        return np.column_stack(self.coords) if self.n else np.empty((0, self.dim))

    def as_tuples(self) -> list:
        return [tuple(float(c[i]) for c in self.coords) for i in range(self.n)]


@dataclass(frozen=True)
class Tolerance:
    """Relative epsilon; the effective length tolerance is eps_rel times the
    input's bounding-box diagonal (geometry.py:68-83).  ``eps_abs`` (not in
    the reference) pins the absolute eps instead -- sharded runs use it so
    every rank and the merge share the global eps."""

    eps_rel: float = DEFAULT_EPS_REL
    eps_abs: float = float("nan")

    def __post_init__(self):
        if self.eps_rel < 0:
            raise ContractViolation("eps_rel must be nonnegative")

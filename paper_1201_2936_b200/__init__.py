"""B200-native Quickhull (Tzeng & Owens, arXiv 1201.2936) behind the hull
entry points of the reference package ``seghull``.

Drop-in names: quickhull_2d, quickhull_3d, HullResult, PointSet, Tolerance,
ContractViolation, EmptyInputError, DegenerateInputError.  Device-tensor
variants: hull_indices_2d, hull_indices_3d.  See DESIGN.md.
"""

from .errors import ContractViolation, DegenerateInputError, EmptyInputError
from .geometry import PointSet, Tolerance
from .quickhull import (HullResult, hull_indices_2d, hull_indices_3d, quickhull_2d, quickhull_3d,
                        trace)

__version__ = "0.1.0"

__all__ = [
    "ContractViolation", "DegenerateInputError", "EmptyInputError", "HullResult", "PointSet",
    "Tolerance", "hull_indices_2d", "hull_indices_3d", "quickhull_2d", "quickhull_3d", "trace",
]

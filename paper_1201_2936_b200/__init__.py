"""B200-native Quickhull (Tzeng & Owens, arXiv 1201.2936) behind the hull
entry points of the reference package ``seghull``.

Drop-in names: quickhull_2d, quickhull_3d, HullResult, PointSet, Tolerance,
ContractViolation, EmptyInputError, DegenerateInputError; the framework
primitives segmented_scan, ScanSpec, flag_permute, compact, scatter,
PermutationMap, head_index_broadcast, segment_ids, reduce_broadcast (GPU ops).
Device-tensor variants: hull_indices_2d, hull_indices_3d (3D facets);
point sources: read_points_device (PTS1 / CSV into HBM), generate_device
(uniform-box clouds generated in HBM); multi-GPU:
paper_1201_2936_b200.sharded.  See DESIGN.md.
"""

from .errors import ContractViolation, DegenerateInputError, EmptyInputError
from .geometry import PointSet, Tolerance
from .primitives import (PermutationMap, ScanSpec, compact, flag_permute, head_index_broadcast,
                         reduce_broadcast, scatter, segment_ids, segmented_scan)
from .quickhull import (HullResult, filter_stats, hull_indices_2d, hull_indices_3d, order_hull_2d,
                        quickhull_2d, quickhull_3d, trace)
from .pointio import PointFileError, generate_device, read_points_device, write_points_binary

__version__ = "0.1.0"

__all__ = [
    "ContractViolation", "DegenerateInputError", "EmptyInputError", "HullResult", "PermutationMap", "filter_stats",
    "PointSet", "ScanSpec", "Tolerance", "compact", "flag_permute", "head_index_broadcast",
    "hull_indices_2d", "hull_indices_3d", "order_hull_2d", "quickhull_2d", "quickhull_3d", "reduce_broadcast",
    "scatter", "segment_ids", "segmented_scan", "trace", "PointFileError", "generate_device",
    "read_points_device", "write_points_binary",
]

"""Drop-in hull entry points backed by the sm_100a CUDA path.

Mirrors the reference drivers' public interface
(/root/reference/pkg/src/seghull/quickhull.py):

  quickhull_2d(points: PointSet, tol: Tolerance = Tolerance()) -> HullResult   (:167)
  quickhull_3d(points: PointSet, tol: Tolerance = Tolerance()) -> HullResult   (:282)
  HullResult(vertices, iterations, discarded, warnings)                         (:34-46)

with the same exceptions (ContractViolation for a dimension mismatch,
EmptyInputError for n = 0, DegenerateInputError for coplanar 3D input,
AssertionError for the round guard) and the same warning strings.  The
vertex coordinates come back in discovery order (first-split extremes, then
round by round); the vertex SET is bit-exact with the reference.

Index-returning variants work on device tensors without a host round trip:

  hull_indices_2d(points) -> int64 CUDA tensor of original point indices
  hull_indices_3d(points) -> (indices, facets or None)

Every call goes through the C ABI (include/seghull_b200.h) into one CUDA
graph launch; there is no CPU fallback.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ContractViolation, DegenerateInputError, EmptyInputError
from .geometry import PointSet, Tolerance


@dataclass
class HullResult:
    """Hull vertex set plus run statistics (reference quickhull.py:34-46).

    ``indices`` (not in the reference) holds the original indices of the
    vertices; ``vertices`` their coordinates in the same order."""

    vertices: PointSet
    iterations: int
    discarded: int
    warnings: list = field(default_factory=list)
    indices: np.ndarray = None
    facets: np.ndarray = None  # 3D, quickhull_3d(..., facets=True): (f, 3) original indices


def _raise_for(rc: int):
    msg = _lib.last_error()
    if rc == _lib.SH_CONTRACT:
        raise ContractViolation(msg)
    if rc == _lib.SH_EMPTY:
        raise EmptyInputError(msg)
    if rc == _lib.SH_DEGENERATE:
        raise DegenerateInputError(msg)
    if rc == _lib.SH_ROUND_GUARD:
        raise AssertionError(msg)
    raise RuntimeError(f"seghull_b200 error {rc}: {msg}")


def _on_host(points):
    first = points[0] if isinstance(points, (tuple, list)) else points
    return torch.is_tensor(first) and first.device.type == "cpu"


def _to_cuda(points):
    """Host tensors (ideally pinned) -> the current CUDA device, async on the
    current stream; the hull launch that follows is ordered after the copy."""
    dev = torch.device("cuda", torch.cuda.current_device())
    if isinstance(points, (tuple, list)):
        return tuple(c.to(dev, non_blocking=True) for c in points)
    return points.to(dev, non_blocking=True)


def _as_device_coords(points, dim):
    """(n, dim) fp64 CUDA tensor (any row stride with unit column stride) or
    a tuple of dim 1-D fp64 CUDA tensors -> (pointers, stride, n, keepalive)."""
    if isinstance(points, (tuple, list)):
        if len(points) != dim:
            raise ContractViolation(f"expected {dim}D points, got {len(points)}D")
        cols = []
        for c in points:
            if not (torch.is_tensor(c) and c.is_cuda and c.dtype == torch.float64 and c.dim() == 1):
                raise ContractViolation("coordinate tensors must be 1-D float64 CUDA tensors")
            cols.append(c.contiguous())
        n = cols[0].numel()
        if any(c.numel() != n for c in cols):
            raise ContractViolation("coordinate arrays must be equal length")
        return [c.data_ptr() for c in cols], 1, n, cols
    t = points
    if not (torch.is_tensor(t) and t.is_cuda and t.dtype == torch.float64 and t.dim() == 2):
        raise ContractViolation("points must be an (n, dim) float64 CUDA tensor")
    if t.shape[1] != dim:
        raise ContractViolation(f"expected {dim}D points, got {t.shape[1]}D")
    if t.stride(1) != 1:
        t = t.contiguous()
    n = t.shape[0]
    base = t.data_ptr()
    return [base + 8 * k for k in range(dim)], t.stride(0), n, [t]


_out_cache = {}


def _out_buffer(device, n):
    """Per-device scratch for the C ABI's index output (capacity n + 2: two
    virtual extremes of a sharded hull); callers copy out the h written
    entries.  Reused across calls (under the device lock) instead of
    allocating 8 bytes per input point every call."""
    buf = _out_cache.get(device)
    if buf is None or buf.numel() < n + 2:
        buf = _out_cache[device] = torch.empty(max(n + 2, 1024), dtype=torch.int64,
                                               device=torch.device("cuda", device))
    return buf


def _stream_ptr(device):
    return torch.cuda.current_stream(device).cuda_stream


class _Shard:
    """sh_set_shard for the duration of one hull call (sharded.py): the whole
    input's statistics (device tensor, SH_STATS doubles), this slice's first
    global index, SH_SHARD_* flags."""

    def __init__(self, shard, ctx):
        self.shard, self.ctx = shard, ctx

    def __enter__(self):
        if self.shard is not None:
            gstats, offset, flags = self.shard
            rc = _lib.lib().sh_set_shard(self.ctx, gstats.data_ptr(), int(offset), int(flags))
            if rc != _lib.SH_OK:
                _raise_for(rc)

    def __exit__(self, *exc):
        if self.shard is not None:
            _lib.lib().sh_set_shard(self.ctx, None, 0, 0)


class _FilterShare:
    """sh_set_filter_share for the duration of one 3D hull call: the filter
    decides only share r of R of the candidates and keeps the others
    (sharded.py's split merge)."""

    def __init__(self, share, ctx):
        self.share, self.ctx = share, ctx

    def __enter__(self):
        if self.share is not None:
            r, R = self.share
            rc = _lib.lib().sh_set_filter_share(self.ctx, int(r), int(R))
            if rc != _lib.SH_OK:
                _raise_for(rc)

    def __exit__(self, *exc):
        if self.share is not None:
            _lib.lib().sh_set_filter_share(self.ctx, 0, 1)


def hull_indices_2d(points, tol: Tolerance = Tolerance(), return_info=False, shard=None):
    """Original indices (int64 tensor) of the 2D hull vertices.

    ``points``: an (n, 2) float64 tensor or a pair of 1-D float64 tensors.
    CUDA input -> CUDA output, no host synchronisation beyond reading the
    vertex count.  Host (CPU, preferably pinned) input is copied to the
    current device first and the indices come back on the host."""
    if _on_host(points):
        r = hull_indices_2d(_to_cuda(points), tol, return_info)
        return (r[0].cpu(), r[1]) if return_info else r.cpu()
    ptrs, stride, n, keep = _as_device_coords(points, 2)
    device = keep[0].device.index
    if n == 0:
        raise EmptyInputError("cannot take the hull of an empty point set")
    res = _lib.ShResult()
    with torch.cuda.device(device), _lib.device_lock(device):
        ctx = _lib.context(device)
        out = _out_buffer(device, n)
        with _Shard(shard, ctx):
            rc = _lib.lib().sh_hull2d(ctx, ptrs[0], ptrs[1], stride, n, tol.eps_rel, tol.eps_abs,
                                      out.data_ptr(), ctypes.byref(res), _stream_ptr(device))
        idx = out[:res.h].clone() if rc == _lib.SH_OK else None
    if rc != _lib.SH_OK:
        _raise_for(rc)
    return (idx, res) if return_info else idx


def hull_indices_3d(points, tol: Tolerance = Tolerance(), facets=False, return_info=False, shard=None,
                    filter_share=None):
    """Original indices (int64 tensor) of the 3D hull vertices, plus the
    (f, 3) int32 facet triples when ``facets`` is true: original indices,
    counter-clockwise seen from outside, exact (coplanar vertices are
    triangulated consistently), order unspecified.  Host input is handled
    like in hull_indices_2d.  ``filter_share`` (r, R): the extreme filter
    decides only share r of R of the candidates and keeps the rest (the
    intersection over the R shares is the hull)."""
    if _on_host(points):
        r = hull_indices_3d(_to_cuda(points), tol, facets, return_info, shard, filter_share)
        if return_info:
            return r[0].cpu(), (None if r[1] is None else r[1].cpu()), r[2]
        return (r[0].cpu(), None if r[1] is None else r[1].cpu()) if facets else r.cpu()
    ptrs, stride, n, keep = _as_device_coords(points, 3)
    device = keep[0].device.index
    if n == 0:
        raise EmptyInputError("cannot take the hull of an empty point set")
    # facets <= 2 * vertices - 4; start from a size that covers volume-like
    # clouds and retry once with the exact count for surface-like ones
    fcap = min(2 * n + 8, max(4096, 16 * int(n ** 0.5))) if facets else 0
    for _ in range(2):
        fout = torch.empty((max(fcap, 1), 3), dtype=torch.int32, device=keep[0].device)
        res = _lib.ShResult()
        with torch.cuda.device(device), _lib.device_lock(device):
            ctx = _lib.context(device)
            out = _out_buffer(device, n)
            with _Shard(shard, ctx), _FilterShare(filter_share, ctx):
                rc = _lib.lib().sh_hull3d(ctx, ptrs[0], ptrs[1], ptrs[2], stride, n, tol.eps_rel,
                                          tol.eps_abs, out.data_ptr(),
                                          fout.data_ptr() if facets else None, fcap,
                                          ctypes.byref(res), _stream_ptr(device))
            idx = out[:res.h].clone() if rc == _lib.SH_OK else None
        if facets and rc == _lib.SH_CONTRACT and res.facets > fcap:
            fcap = int(res.facets)
            continue
        break
    if rc != _lib.SH_OK:
        _raise_for(rc)
    fac = fout[:res.facets] if facets else None
    if return_info:
        return idx, fac, res
    return (idx, fac) if facets else idx


def trace(device=None):
    """Per-round counters of the last hull on ``device``: rows of (live points
    entering, survivors, segments, near-coplanar segments dropped)."""
    device = torch.cuda.current_device() if device is None else device
    cap = 4096
    arrs = [np.zeros(cap, np.int64) for _ in range(4)]
    with _lib.device_lock(device):
        r = _lib.lib().sh_trace(_lib.context(device), *(a.ctypes.data for a in arrs), cap)
    return np.stack([a[:r] for a in arrs], axis=1)


def hull_warnings(dim, res, trace_rows=None):
    """The reference's warning strings for a hull result (quickhull.py:208,
    :308-310, :338, :387-389); ``trace_rows``: trace() of the same hull (3D
    per-round near-coplanar drops)."""
    warnings = []
    if res.flags & _lib.SH_FLAG_COLLINEAR:
        warnings.append("collinear input: hull is the two x-extrema" if dim == 2
                        else "collinear input: hull is the two extrema")  # :208 / :338
    if dim == 3:
        if trace_rows is not None and res.iterations:
            for r, (_, _, _, flat) in enumerate(trace_rows, start=1):
                if flat:
                    warnings.append(f"round {r}: dropped {int(flat)} near-coplanar segment(s)")  # :387-389
        if res.pruned:
            warnings.append(f"pruned {int(res.pruned)} non-extreme candidate vertex(es) emitted by "
                            "incomplete per-face outside sets")  # :308-310
    return warnings


FILTER_STATS = ("candidates", "grid", "ambiguous", "gjk_capped", "certified", "queries", "scanned",
                "gjk_iters", "local_pruned", "local_extreme", "global_gjk", "cyc_cert", "cyc_local",
                "cyc_query", "cyc_global") + tuple(f"item_cyc_2^{10 + k}" for k in range(20)) + (
                "item_cyc_max", "item_max_iters", "item_max_queries", "item_max_scanned")


def filter_stats(device=None):
    """Diagnostics of the last 3D extreme filter on ``device`` (sh_filter_stats):
    ``ambiguous`` counts candidates kept because they lie within eps of the
    other candidates' hull boundary, ``gjk_capped`` those whose GJK hit its
    iteration cap (both 0 on inputs in general position)."""
    device = torch.cuda.current_device() if device is None else device
    out = np.zeros(len(FILTER_STATS), np.int64)
    with _lib.device_lock(device):
        k = _lib.lib().sh_filter_stats(_lib.context(device), out.ctypes.data, len(out))
    return dict(zip(FILTER_STATS[:k], out[:k].tolist()))


def _validate(points: PointSet, dim: int):
    # quickhull.py:103-107
    if points.dim != dim:
        raise ContractViolation(f"expected {dim}D points, got {points.dim}D")
    if points.n == 0:
        raise EmptyInputError("cannot take the hull of an empty point set")


def _to_device(points: PointSet):
    dev = torch.device("cuda", torch.cuda.current_device())
    return tuple(torch.from_numpy(c).to(dev, non_blocking=False) for c in points.coords)


def quickhull_2d(points: PointSet, tol: Tolerance = Tolerance()) -> HullResult:
    """Strict 2D hull (reference quickhull.py:167-279), computed on the GPU."""
    _validate(points, 2)
    cols = _to_device(points)
    idx, res = hull_indices_2d(cols, tol, return_info=True)
    idx = idx.cpu().numpy()
    verts = PointSet(tuple(c[idx] for c in points.coords))
    return HullResult(verts, int(res.iterations), points.n - verts.n, hull_warnings(2, res), idx)


def order_hull_2d(vertices: PointSet) -> PointSet:
    """CCW boundary order of a convex vertex set, starting at the
    lexicographically smallest vertex (reference quickhull.py:449-461: angle
    sort around the centroid, stable), computed on the GPU (sh_order_hull_2d:
    centroid, atan2 keys, stable radix sort, rotation).  The result equals
    the reference's order whenever no two vertices share an angle from the
    centroid (always, for a strictly convex set)."""
    if vertices.dim != 2:
        raise ContractViolation("order_hull_2d needs 2D points")
    if vertices.n < 3:
        return vertices
    device = torch.cuda.current_device()
    x, y = (torch.from_numpy(np.ascontiguousarray(c)).to(torch.device("cuda", device))
            for c in vertices.coords)
    perm = torch.empty(vertices.n, dtype=torch.int64, device=x.device)
    with torch.cuda.device(device), _lib.device_lock(device):
        rc = _lib.lib().sh_order_hull_2d(_lib.context(device), x.data_ptr(), y.data_ptr(), vertices.n,
                                         perm.data_ptr(), _stream_ptr(device))
    if rc != _lib.SH_OK:
        _raise_for(rc)
    p = perm.cpu().numpy()
    return PointSet(tuple(np.ascontiguousarray(c[p]) for c in vertices.coords))


def giftwrap_2d(points, eps: float):
    """Indices of the strict 2D hull by gift wrapping on the device, in CCW
    order from the lexicographic minimum (the reference's brute-force check,
    hull2_giftwrap in the reference seghull/oracle module lines 20-52, used by the CLI's `verify`).  ``points``: (n, 2) float64
    CUDA tensor."""
    n = points.shape[0]
    device = points.device.index
    x, y = points[:, 0].contiguous(), points[:, 1].contiguous()
    out = torch.empty(n + 1, dtype=torch.int64, device=points.device)
    h = ctypes.c_int64(0)
    with torch.cuda.device(device), _lib.device_lock(device):
        rc = _lib.lib().sh_giftwrap_2d(_lib.context(device), x.data_ptr(), y.data_ptr(), n, float(eps),
                                       out.data_ptr(), n + 1, ctypes.byref(h), _stream_ptr(device))
    if rc != _lib.SH_OK:
        _raise_for(rc)
    return out[:h.value]


def quickhull_3d(points: PointSet, tol: Tolerance = Tolerance(), facets: bool = False) -> HullResult:
    """3D hull vertex set (reference quickhull.py:282-446), computed on the
    GPU.  ``facets=True`` (not in the reference) also fills
    ``HullResult.facets`` with the hull's triangles."""
    _validate(points, 3)
    cols = _to_device(points)
    device = cols[0].device.index
    with _lib.device_lock(device):  # the hull and its trace, as one unit
        idx, fac, res = hull_indices_3d(cols, tol, facets=facets, return_info=True)
        tr = trace(device) if res.iterations else None
    idx = idx.cpu().numpy()
    warnings = hull_warnings(3, res, tr)
    verts = PointSet(tuple(c[idx] for c in points.coords)) if idx.size else PointSet.empty(3)
    return HullResult(verts, int(res.iterations), points.n - verts.n, warnings, idx,
                      fac.cpu().numpy() if fac is not None else None)

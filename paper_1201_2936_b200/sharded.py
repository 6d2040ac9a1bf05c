"""Sharded Quickhull across GPUs.

The point cloud is split into contiguous index slices, one per rank (one
process per GPU).  The ranks exchange only small messages:

  1. every rank computes its slice's bounding box on the device (sh_bbox);
     an all-reduce (MIN / MAX) gives the whole input's box, and every rank
     derives the same eps = eps_rel * hypot.reduce(spans), which is exactly
     the reference's Tolerance.effective of the whole input
     (geometry.py:79-83);
  2. every rank hulls its slice on its own GPU with that eps (the full
     single-GPU path, 3D extreme filter included);
  3. an all-gather of (count) and then of the padded candidate records
     (coordinates + global index) brings the per-rank hull vertices to
     every rank;
  4. rank 0 hulls the union, with the same eps, after sorting it by global
     index so that the "lowest original index" tie-breaks see the global
     order.

hull(all) = hull(union of the shard hulls), so the vertex set equals the
single-GPU one for inputs in general position (SURVEY.md Appendix A.7 checked
disk, near-circle, square, ball and cube).  The on-circle config (C3) keeps
path-dependent eps decisions and must not be sharded.

The exchanged data is tiny (48 B of box, ~10^4-10^5 records of 32 B), so
the collectives are latency-bound NCCL calls over NVLink; the hull work has
no collective inside it.  The same code runs over gloo on CPU tensors (tests)
and in a single-process "loopback" mode that hulls P slices one after the
other on one GPU (tests, and P-way checking on a 1-GPU box).
"""

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .geometry import Tolerance


def hypot_reduce(spans):
    """np.hypot.reduce(spans) with the library's glibc-exact hypot port
    (hypot.reduce([a, b, c]) == hypot(hypot(a, b), c) bitwise)."""
    acc = float(spans[0])
    for s in spans[1:]:
        a = np.array([acc]), np.array([float(s)]), np.zeros(1)
        _lib.lib().sh_hypot_host(a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data, 1)
        acc = float(a[2][0])
    return acc


def effective_eps(lo, hi, tol: Tolerance):
    """Tolerance.effective from a (global) bounding box."""
    if not math.isnan(tol.eps_abs):
        return tol.eps_abs
    spans = [float(h) - float(l) for l, h in zip(lo, hi)]
    return tol.eps_rel * hypot_reduce(spans)


def _columns(points):
    if isinstance(points, (tuple, list)):
        return tuple(points)
    return tuple(points[:, k] for k in range(points.shape[1]))


def device_bbox(cols):
    """(2*dim,) float64 device tensor: per-axis min then max (own kernel)."""
    dim = len(cols)
    dev = cols[0].device
    out = torch.empty(2 * dim, dtype=torch.float64, device=dev)
    cc = [c.contiguous() if c.stride(0) != cols[0].stride(0) else c for c in cols]
    stride = cc[0].stride(0)
    with torch.cuda.device(dev):
        rc = _lib.lib().sh_bbox(_lib.context(dev.index), cc[0].data_ptr(), cc[1].data_ptr(),
                                cc[2].data_ptr() if dim == 3 else None, stride, cc[0].numel(), dim,
                                out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    if rc != _lib.SH_OK:
        raise RuntimeError(f"sh_bbox failed ({rc}): {_lib.last_error()}")
    return out


def device_hull(cols, tol: Tolerance):
    """Local hull of one slice on its GPU (the product path)."""
    from .quickhull import hull_indices_2d, hull_indices_3d
    if len(cols) == 2:
        return hull_indices_2d(tuple(cols), tol)
    return hull_indices_3d(tuple(cols), tol)


def _records(cols, idx, offset):
    """Candidate records: coordinates + global index (exact in fp64 below 2^53)."""
    parts = [c[idx] for c in cols] + [(idx + offset).to(torch.float64)]
    return torch.stack(parts, dim=1)


def _merge(union, dim, eps_rel, eps, local_hull):
    """Final hull of the gathered records; returns global indices."""
    if union.shape[0] == 0:
        return torch.empty(0, dtype=torch.int64, device=union.device)
    union = union[torch.argsort(union[:, dim])]  # global index order
    cols = tuple(union[:, k].contiguous() for k in range(dim))
    fidx = local_hull(cols, Tolerance(eps_rel, eps_abs=eps))
    return union[fidx.to(union.device), dim].to(torch.int64)


def hull_sharded(points, offset, tol: Tolerance = Tolerance(), group=None, local_hull=None,
                 local_bbox=None, return_info=False):
    """Hull of a point cloud sharded over the ranks of ``group``.

    points: this rank's slice, an (n_i, dim) float64 tensor or a tuple of dim
    1-D tensors (CUDA for the product path / NCCL; CPU with gloo when
    ``local_hull`` and ``local_bbox`` are given).  offset: global index of
    the slice's first point.  Returns the global vertex indices (int64) on
    rank 0 and None on the other ranks.
    """
    import torch.distributed as dist
    cols = _columns(points)
    dim = len(cols)
    local_hull = local_hull or device_hull
    local_bbox = local_bbox or device_bbox
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = cols[0].device
    # 1. global bounding box -> identical eps on every rank
    if cols[0].numel():
        bb = local_bbox(cols)
    else:
        bb = torch.tensor([math.inf] * dim + [-math.inf] * dim, dtype=torch.float64, device=dev)
    lo, hi = bb[:dim].clone(), bb[dim:].clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    lo_h, hi_h = lo.cpu().tolist(), hi.cpu().tolist()
    eps = effective_eps(lo_h, hi_h, tol)
    # 2. local hull with the global eps
    if cols[0].numel():
        idx = local_hull(cols, Tolerance(tol.eps_rel, eps_abs=eps)).to(dev)
    else:
        idx = torch.empty(0, dtype=torch.int64, device=dev)
    rec = _records(cols, idx, offset)
    # 3. all-gather the candidate records (counts first, then padded rows)
    cnt = torch.tensor([rec.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(max(counts), 1)
    pad = torch.zeros((cap, dim + 1), dtype=torch.float64, device=dev)
    pad[:rec.shape[0]] = rec
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    # 4. rank 0: hull of the union
    result = None
    if rank == 0:
        union = torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
        result = _merge(union, dim, tol.eps_rel, eps, local_hull)
    if return_info:
        return result, {"eps": eps, "local_candidates": counts, "union": sum(counts)}
    return result


def hull_sharded_loopback(points, nshards, tol: Tolerance = Tolerance(), local_hull=None,
                          local_bbox=None, return_info=False):
    """The same shard -> merge pipeline for ``nshards`` contiguous slices in
    one process (collectives replaced by their obvious local equivalents)."""
    cols = _columns(points)
    dim = len(cols)
    n = cols[0].numel()
    local_hull = local_hull or device_hull
    local_bbox = local_bbox or device_bbox
    bounds = [(n * r) // nshards for r in range(nshards + 1)]
    slices = [tuple(c[bounds[r]:bounds[r + 1]] for c in cols) for r in range(nshards)]
    boxes = [local_bbox(s) for s in slices if s[0].numel()]
    lo = torch.stack([b[:dim] for b in boxes]).min(dim=0).values.cpu().tolist()
    hi = torch.stack([b[dim:] for b in boxes]).max(dim=0).values.cpu().tolist()
    eps = effective_eps(lo, hi, tol)
    recs = []
    for r, s in enumerate(slices):
        if s[0].numel() == 0:
            continue
        idx = local_hull(s, Tolerance(tol.eps_rel, eps_abs=eps)).to(cols[0].device)
        recs.append(_records(s, idx, bounds[r]))
    union = torch.cat(recs, dim=0)
    result = _merge(union, dim, tol.eps_rel, eps, local_hull)
    if return_info:
        return result, {"eps": eps, "local_candidates": [r.shape[0] for r in recs], "union": union.shape[0]}
    return result

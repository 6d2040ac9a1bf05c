"""Sharded Quickhull across GPUs.

The point cloud is split into contiguous index slices, one per rank (one
process per GPU).  The ranks exchange only small messages, and the host
waits for the device only where a size must be known:

  1. every rank runs one statistics pass over its slice on the device
     (sh_stats: bounding box and lexicographic extremes with global indices,
     quickhull.py:75-84); ONE all-gather (NCCL over NVLink) of these
     14-double records, reduced on the device (sh_stats_reduce), gives every
     rank the whole input's box and extreme points;
  2. every rank hulls its slice with them, read on the device
     (sh_set_shard): eps = eps_rel * hypot.reduce(global spans) -- exactly
     the reference's Tolerance.effective of the whole input
     (geometry.py:79-83) -- and the first split along the global extremes
     (hull vertices of the whole input, entering slices that do not hold them
     as virtual points), so every rank discards what the whole input's first
     split discards; the full single-GPU path, 3D extreme filter included;
  3. one all-gather of (candidate count, status) -- a rank whose slice is
     degenerate (3D coplanar) contributes all its points, any other failure
     is raised on every rank instead of leaving the others blocked in a
     collective -- then an all-gather of the padded candidate records
     (coordinates + global index);
  4. rank 0 hulls the union, deduplicated and sorted by global index so that
     the "lowest original index" tie-breaks see the global order, with the
     same eps.

hull(all) = hull(union of the shard hulls), so the vertex set equals the
single-GPU one for inputs in general position (SURVEY.md Appendix A.7 checked
disk, near-circle, square, ball and cube).  The on-circle config (C3) keeps
path-dependent eps decisions and must not be sharded.

The same code runs over gloo on CPU tensors (tests, with CPU stand-ins for the
device statistics and hull) and in a single-process "loopback" mode that
hulls P slices one after the other on one GPU (tests, and P-way checking on a
1-GPU box).
"""

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .errors import DegenerateInputError
from .geometry import Tolerance

STATS = _lib.SH_STATS


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


def eps_of_stats(gstats, dim, tol: Tolerance):
    """Tolerance.effective of the whole input from reduced statistics (host)."""
    g = gstats.cpu().numpy()
    return effective_eps(-g[:dim], g[3:3 + dim], tol)


def _columns(points):
    if isinstance(points, (tuple, list)):
        return tuple(points)
    return tuple(points[:, k] for k in range(points.shape[1]))


def _contiguous(cols):
    """Unit-stride columns (the C ABI takes one element stride for all of
    them)."""
    return tuple(c if c.stride(0) == 1 else c.contiguous() for c in cols)


def empty_stats(dim, device):
    """Statistics of an empty slice: neutral for the reduction."""
    s = torch.full((STATS,), -math.inf, dtype=torch.float64, device=device)
    s[6:9] = math.inf   # lex-min record: larger than everything
    s[9] = math.inf
    if dim == 2:
        s[2] = s[5] = 0.0
    return s


def device_stats(cols, offset):
    """(SH_STATS,) float64 device tensor: sh_stats of this slice (one pass,
    stream-ordered)."""
    cols = _contiguous(cols)
    dim = len(cols)
    dev = cols[0].device
    out = torch.empty(STATS, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        rc = _lib.lib().sh_stats(_lib.context(dev.index), cols[0].data_ptr(), cols[1].data_ptr(),
                                 cols[2].data_ptr() if dim == 3 else None, 1, cols[0].numel(), dim,
                                 int(offset), out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    if rc != _lib.SH_OK:
        raise RuntimeError(f"sh_stats failed ({rc}): {_lib.last_error()}")
    return out


def device_reduce_stats(gathered, dim):
    """(world, SH_STATS) device tensor -> the whole input's statistics."""
    gathered = gathered.contiguous()
    dev = gathered.device
    out = torch.empty(STATS, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        rc = _lib.lib().sh_stats_reduce(_lib.context(dev.index), gathered.data_ptr(), gathered.shape[0], dim,
                                        out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    if rc != _lib.SH_OK:
        raise RuntimeError(f"sh_stats_reduce failed ({rc}): {_lib.last_error()}")
    return out


def device_bbox(cols):
    """(2*dim,) float64 device tensor: per-axis min then max (own kernel)."""
    dim = len(cols)
    s = device_stats(cols, 0)
    return torch.cat([-s[:dim], s[3:3 + dim]])


def device_hull(cols, offset, tol: Tolerance, gstats):
    """Local hull of one slice on its GPU (the product path) with the whole
    input's statistics: global eps and first-split extremes read on the
    device.  Returns (global indices, coordinates (k, dim), eps used)."""
    from .quickhull import hull_indices_2d, hull_indices_3d
    cols = _contiguous(cols)
    dim, n = len(cols), cols[0].numel()
    flags = _lib.SH_SHARD_SPLIT | (_lib.SH_SHARD_EPS if math.isnan(tol.eps_abs) else 0)
    shard = (gstats, offset, flags)
    if dim == 2:
        idx, res = hull_indices_2d(cols, tol, return_info=True, shard=shard)
    else:
        idx, _, res = hull_indices_3d(cols, tol, return_info=True, shard=shard)
    # virtual points n (global lex-min) and n + 1 (global lex-max): their
    # records come from the statistics
    return _globalize(cols, offset, idx, gstats) + (float(res.eps),)


class StagedDeviceHull:
    """The product path of one rank: the local hull in two halves around the
    statistics exchange (sh_hull_shard_begin / _end), so the statistics come
    from the hull's own first pass instead of an extra pass over the slice.
    The device's context is held from begin() to end()."""

    def __init__(self):
        self.lock = None

    def begin(self, cols, offset, tol: Tolerance):
        cols = _contiguous(cols)
        self.cols, self.offset, self.tol = cols, offset, tol
        dev = cols[0].device
        self.device = dev.index
        out = torch.empty(STATS, dtype=torch.float64, device=dev)
        self.lock = _lib.device_lock(self.device)
        self.lock.acquire()
        try:
            with torch.cuda.device(dev):
                dim = len(cols)
                rc = _lib.lib().sh_hull_shard_begin(
                    _lib.context(self.device), dim, cols[0].data_ptr(), cols[1].data_ptr(),
                    cols[2].data_ptr() if dim == 3 else None, 1, cols[0].numel(), tol.eps_rel, tol.eps_abs,
                    int(offset), out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
            if rc != _lib.SH_OK:
                from .quickhull import _raise_for
                _raise_for(rc)
        except BaseException:
            self.release()
            raise
        return out

    def end(self, cols, offset, tol, gstats):
        from .quickhull import _out_buffer, _raise_for
        try:
            dim, n = len(self.cols), self.cols[0].numel()
            flags = _lib.SH_SHARD_SPLIT | (_lib.SH_SHARD_EPS if math.isnan(tol.eps_abs) else 0)
            res = _lib.ShResult()
            dev = self.cols[0].device
            with torch.cuda.device(dev):
                out = _out_buffer(self.device, n)
                rc = _lib.lib().sh_hull_shard_end(_lib.context(self.device), gstats.data_ptr(), flags,
                                                  out.data_ptr(), ctypes.byref(res),
                                                  torch.cuda.current_stream(dev).cuda_stream)
                if rc != _lib.SH_OK:
                    _raise_for(rc)
                idx = out[:res.h].clone()
        finally:
            self.release()
        return _globalize(self.cols, self.offset, idx, gstats) + (float(res.eps),)

    def release(self):
        if self.lock is not None:
            self.lock.release()
            self.lock = None


def _globalize(cols, offset, idx, gstats):
    """Local hull indices (n, n + 1: the virtual global extremes) -> global
    indices and coordinates (k, dim)."""
    dim, n = len(cols), cols[0].numel()
    virt = idx >= n
    coords = torch.stack([c[torch.where(virt, torch.zeros_like(idx), idx)] for c in cols], dim=1)
    gidx = idx + offset
    if bool(virt.any()):
        vrec = gstats[6:].view(2, 4)[(idx - n).clamp(0, 1)]
        coords = torch.where(virt[:, None], vrec[:, :dim], coords)
        gidx = torch.where(virt, vrec[:, 3].to(torch.int64), gidx)
    return gidx, coords


def device_merge_hull(cols, tol: Tolerance, share=None):
    """The hull of the union (plain hull: the union holds the global extremes
    as real points; tol carries the global eps).  share (r, R): in 3D the
    extreme filter decides only share r of R of the candidates and keeps the
    others (the split merge of hull_sharded)."""
    from .quickhull import hull_indices_2d, hull_indices_3d
    cols = _contiguous(cols)
    if len(cols) == 2:
        return hull_indices_2d(cols, tol)
    return hull_indices_3d(cols, tol, filter_share=share)


def _local(cols, offset, tol, gstats, local_hull, device):
    """(records (k, dim + 1), status, eps, message) of this slice: status 0
    ok, 1 the slice is degenerate (all its points are sent), 2 failure."""
    dim, n = len(cols), cols[0].numel()
    if n == 0:
        return torch.zeros((0, dim + 1), dtype=torch.float64, device=device), 0, math.nan, ""
    try:
        gidx, coords, eps = local_hull(cols, offset, tol, gstats)
        return torch.cat([coords, gidx.to(torch.float64)[:, None]], dim=1), 0, eps, ""
    except DegenerateInputError:
        # a coplanar slice: its points all stay candidates of the merge
        allp = torch.stack(list(cols) + [torch.arange(offset, offset + n, dtype=torch.float64,
                                                      device=device)], dim=1)
        return allp, 1, math.nan, ""
    except Exception as e:  # reported on every rank, see hull_sharded
        return torch.zeros((0, dim + 1), dtype=torch.float64, device=device), 2, math.nan, repr(e)


def _merge(union, dim, eps, merge_hull, share=None):
    """Final hull of the gathered records (deduplicated, in global index
    order); returns global indices.  share: see device_merge_hull."""
    if union.shape[0] == 0:
        return torch.empty(0, dtype=torch.int64, device=union.device)
    union = union[torch.argsort(union[:, dim])]
    keep = torch.ones(union.shape[0], dtype=torch.bool, device=union.device)
    keep[1:] = union[1:, dim] != union[:-1, dim]  # a global extreme comes from every slice
    union = union[keep]
    cols = tuple(union[:, k].contiguous() for k in range(dim))
    t = Tolerance(eps_abs=eps)
    idx = merge_hull(cols, t) if share is None else merge_hull(cols, t, share=share)
    return union[idx.to(union.device), dim].to(torch.int64)


def _all_gather(t, group):
    """(world, *t.shape) tensor of every rank's ``t`` (one collective)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return torch.stack(parts)


def _single_rank(cols, offset, tol, return_info):
    """hull_sharded on a one-rank group: the plain device hull, its indices
    shifted by the slice offset; failures raise as from the protocol."""
    from .quickhull import hull_indices_2d, hull_indices_3d
    cols = _contiguous(cols)
    dim, n = len(cols), cols[0].numel()
    if n == 0:
        idx, eps = torch.empty(0, dtype=torch.int64, device=cols[0].device), math.nan
    else:
        try:
            if dim == 2:
                idx, res = hull_indices_2d(cols, tol, return_info=True)
            else:
                idx, _, res = hull_indices_3d(cols, tol, return_info=True)
        except DegenerateInputError:
            raise
        except Exception as e:
            raise RuntimeError(f"sharded hull failed on rank(s) [0]: {e!r}") from e
        idx, eps = idx + offset, float(res.eps)
    if return_info:
        return idx, {"eps": eps, "local_candidates": [idx.numel()], "union": idx.numel()}
    return idx


def hull_sharded(points, offset, tol: Tolerance = Tolerance(), group=None, local_hull=None,
                 local_stats=None, reduce_stats=None, merge_hull=None, return_info=False,
                 split_merge=None):
    """Hull of a point cloud sharded over the ranks of ``group``.

    points: this rank's slice, an (n_i, dim) float64 tensor or a tuple of dim
    1-D tensors (CUDA for the product path / NCCL; CPU with gloo when the
    stand-ins ``local_hull``, ``local_stats``, ``reduce_stats`` and
    ``merge_hull`` are given).  offset: global index of the slice's first
    point.  Returns the global vertex indices (int64) on rank 0 and None on
    the other ranks; every rank raises if any rank failed.  split_merge (3D;
    default: on for the product path): every rank runs the merge loop on the
    gathered union and decides the extreme filter for its share of the
    candidates; rank 0 intersects the vertex lists (one more all-gather).
    """
    import torch.distributed as dist
    cols = _columns(points)
    dim = len(cols)
    if (local_hull is None and local_stats is None and merge_hull is None
            and dist.get_world_size(group) == 1):
        # one rank: the slice is the whole input, so the global statistics
        # are its own and the protocol reduces to the plain hull -- run that
        # (no exchange, one graph launch)
        return _single_rank(cols, offset, tol, return_info)
    staged = None
    if local_hull is None and local_stats is None:
        # the product path: the statistics come from the hull's own first pass
        staged = StagedDeviceHull()
        local_stats = lambda c, o: staged.begin(c, o, tol)
        local_hull = staged.end
    local_hull = local_hull or device_hull
    local_stats = local_stats or device_stats
    reduce_stats = reduce_stats or device_reduce_stats
    merge_hull = merge_hull or device_merge_hull
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = cols[0].device
    # 1. statistics of every slice, one all-gather, reduced on the device
    begun = True
    try:
        st = local_stats(cols, offset) if cols[0].numel() else empty_stats(dim, dev)
    except Exception as e:  # still take part in the exchange; reported below
        st, begun, msg0 = empty_stats(dim, dev), False, repr(e)
    try:
        gstats = reduce_stats(_all_gather(st, group), dim)
    except BaseException:
        if staged:
            staged.release()
        raise
    # 2. local hull with the global eps and first split (device-side)
    if begun:
        rec, status, eps, msg = _local(cols, offset, tol, gstats, local_hull, dev)
    else:
        rec, status, eps, msg = torch.zeros((0, dim + 1), dtype=torch.float64, device=dev), 2, math.nan, msg0
    if staged:
        staged.release()
    if world == 1:  # the slice is the whole input: its hull is the answer
        if status == 2:
            raise RuntimeError(f"sharded hull failed on rank(s) [0]: {msg}")
        if status == 1:  # degenerate: the single hull raises the same error
            merge_hull(cols, tol)
        result = rec[:, dim].to(torch.int64)
        if return_info:
            return result, {"eps": eps, "local_candidates": [rec.shape[0]], "union": rec.shape[0]}
        return result
    # 3. candidate counts and status, then the records
    cs = torch.tensor([rec.shape[0], status], dtype=torch.int64, device=dev)
    allcs = _all_gather(cs, group).cpu().tolist()  # the one host read of the exchange
    if any(s == 2 for _, s in allcs):
        bad = [r for r, (_, s) in enumerate(allcs) if s == 2]
        raise RuntimeError(f"sharded hull failed on rank(s) {bad}" + (f": {msg}" if msg else ""))
    counts = [c for c, _ in allcs]
    cap = max(max(counts), 1)
    pad = torch.zeros((cap, dim + 1), dtype=torch.float64, device=dev)
    pad[:rec.shape[0]] = rec
    parts = _all_gather(pad, group)
    # 4. hull of the union: on rank 0, or (3D, split) the loop on every rank
    # with the filter split over the ranks, the vertex lists intersected
    if split_merge is None:
        split_merge = merge_hull is device_merge_hull
    split = split_merge and dim == 3
    result = None
    if rank == 0 or split:
        if math.isnan(eps):
            eps = eps_of_stats(gstats, dim, tol)
        union = torch.cat([parts[r, :c] for r, c in enumerate(counts)], dim=0)
        if not split:
            result = _merge(union, dim, eps, merge_hull)
        else:
            mine = _merge(union, dim, eps, merge_hull, share=(rank, world))
            lens = _all_gather(torch.tensor([mine.numel()], dtype=torch.int64, device=dev), group)
            lens = lens.view(-1).cpu().tolist()
            padk = torch.full((max(max(lens), 1),), -1, dtype=torch.int64, device=dev)
            padk[:mine.numel()] = mine.to(dev)
            allk = _all_gather(padk, group)
            if rank == 0:
                keep = torch.ones(mine.numel(), dtype=torch.bool, device=dev)
                for r in range(1, world):
                    keep &= torch.isin(padk[:mine.numel()], allk[r, :lens[r]])
                result = mine.to(dev)[keep]
    if return_info:
        return result, {"eps": eps, "local_candidates": counts, "union": sum(counts)}
    return result


def hull_sharded_loopback(points, nshards, tol: Tolerance = Tolerance(), local_hull=None,
                          local_stats=None, reduce_stats=None, merge_hull=None, return_info=False,
                          split_merge=None):
    """The same shard -> merge pipeline for ``nshards`` contiguous slices in
    one process (collectives replaced by their obvious local equivalents;
    the split 3D merge runs its shares one after the other)."""
    cols = _columns(points)
    dim = len(cols)
    n = cols[0].numel()
    dev = cols[0].device
    local_hull = local_hull or device_hull
    local_stats = local_stats or device_stats
    reduce_stats = reduce_stats or device_reduce_stats
    merge_hull = merge_hull or device_merge_hull
    bounds = [(n * r) // nshards for r in range(nshards + 1)]
    slices = [tuple(c[bounds[r]:bounds[r + 1]] for c in cols) for r in range(nshards)]
    stats = [local_stats(s, bounds[r]) if s[0].numel() else empty_stats(dim, dev)
             for r, s in enumerate(slices)]
    gstats = reduce_stats(torch.stack(stats), dim)
    recs, eps = [], math.nan
    for r, s in enumerate(slices):
        rec, status, e, msg = _local(s, bounds[r], tol, gstats, local_hull, dev)
        if status == 2:
            raise RuntimeError(f"sharded hull failed on slice {r}: {msg}")
        eps = e if math.isnan(eps) else eps
        recs.append(rec)
    if math.isnan(eps):
        eps = eps_of_stats(gstats, dim, tol)
    union = torch.cat(recs, dim=0)
    if split_merge is None:
        split_merge = merge_hull is device_merge_hull
    if split_merge and dim == 3 and nshards > 1:
        lists = [_merge(union, dim, eps, merge_hull, share=(r, nshards)) for r in range(nshards)]
        keep = torch.ones(lists[0].numel(), dtype=torch.bool, device=lists[0].device)
        for other in lists[1:]:
            keep &= torch.isin(lists[0], other)
        result = lists[0][keep]
    else:
        result = _merge(union, dim, eps, merge_hull)
    if return_info:
        return result, {"eps": eps, "local_candidates": [r.shape[0] for r in recs], "union": union.shape[0]}
    return result

"""Sharded hull host logic: bbox all-reduce -> global eps,
per-rank hull, all-gather of candidate records, rank-0 merge.

CPU tests run the real distributed code over gloo with world_size 2; the
per-rank hull is the CPU oracle standing in for the device (the checker
used as a mock of the GPU kernel -- the product's default local hull is
the CUDA path).  The GPU tests run the same pipeline with the device hull
in loopback mode (P slices on one GPU)."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1201_2936_b200 import sharded
from paper_1201_2936_b200.datagen import generate
from paper_1201_2936_b200.errors import DegenerateInputError
from paper_1201_2936_b200.geometry import Tolerance


def cpu_stats(cols, offset):
    """Host stand-in for sh_stats: -lo, hi (z = 0 in 2D), lexicographic
    min / max records (x, y, z, global index), lowest index among ties for
    the min, highest for the max (quickhull.py:75-84)."""
    a = [c.numpy() for c in cols]
    dim = len(a)
    s = np.zeros(14)
    for k in range(dim):
        s[k], s[3 + k] = -a[k].min(), a[k].max()
    keys = tuple(reversed(a))  # np.lexsort: last key is primary
    order = np.lexsort(keys)
    mn = order[0]
    mx = order[-1]
    # highest index among full ties for the max
    ties = np.flatnonzero(np.all([c == c[mx] for c in a], axis=0))
    mx = ties.max()
    for k in range(dim):
        s[6 + k], s[10 + k] = a[k][mn], a[k][mx]
    s[9], s[13] = offset + mn, offset + mx
    return torch.from_numpy(s)


def cpu_reduce_stats(gathered, dim):
    g = gathered.numpy()
    out = g[0].copy()
    out[:6] = g[:, :6].max(axis=0)
    key = lambda r: tuple(r[:dim]) + (r[3],)
    out[6:10] = min((r[6:10] for r in g), key=key)
    out[10:14] = max((r[10:14] for r in g), key=key)
    return torch.from_numpy(out)


def cpu_hull(cols, offset, tol, gstats):
    """Oracle stand-in for the device hull of a slice (exact reference
    semantics, with the whole input's eps)."""
    dim = len(cols)
    eps = sharded.eps_of_stats(gstats, dim, tol)
    arrs = [c.numpy() for c in cols]
    if dim == 2:
        idx = oracle.hull2d(*arrs, eps_rel=tol.eps_rel, eps_abs=eps).idx
    else:
        r, idx, _ = oracle.full_hull3d(*arrs, eps_rel=tol.eps_rel, eps_abs=eps)
        if r.status == oracle.STATUS_DEGENERATE:
            raise DegenerateInputError("all points are coplanar")
    idx = torch.from_numpy(np.asarray(idx, dtype=np.int64).copy())
    coords = torch.stack([c[idx] for c in cols], dim=1)
    return idx + offset, coords, eps


def cpu_merge(cols, tol):
    arrs = [c.numpy() for c in cols]
    if len(arrs) == 2:
        return torch.from_numpy(oracle.hull2d(*arrs, eps_rel=tol.eps_rel, eps_abs=tol.eps_abs).idx.copy())
    idx = oracle.full_hull3d(*arrs, eps_rel=tol.eps_rel, eps_abs=tol.eps_abs)[1]
    return torch.from_numpy(np.asarray(idx, dtype=np.int64).copy())


CPU = dict(local_hull=cpu_hull, local_stats=cpu_stats, reduce_stats=cpu_reduce_stats, merge_hull=cpu_merge)


def cpu_merge_share(cols, tol, share=None):
    """Stand-in for the split merge (3D): share r of R returns the hull plus
    the union points whose position is not congruent to r mod R -- like the
    device filter, which keeps every candidate outside its share; only the
    intersection over the shares is the hull."""
    exact = cpu_merge(cols, tol)
    if share is None:
        return exact
    r, R = share
    n = cols[0].numel()
    extra = torch.tensor([p for p in range(n) if p % R != r], dtype=torch.int64)
    extra = extra[~torch.isin(extra, exact)]
    return torch.cat([exact, extra])


def _split_worker(rank, world, port, kind, n, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cols = generate(kind, n, 0)
    b = [(n * r) // world for r in range(world + 1)]
    mine = tuple(torch.from_numpy(np.ascontiguousarray(c[b[rank]:b[rank + 1]])) for c in cols)
    hooks = dict(CPU, merge_hull=cpu_merge_share)
    res = sharded.hull_sharded(mine, b[rank], Tolerance(), split_merge=True, **hooks)
    q.put((rank, None if res is None else np.sort(res.numpy())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_split_merge_intersects_shares(world):
    """3D merge split over the ranks (every rank runs the merge with its
    filter share, rank 0 intersects): the whole input's hull on rank 0."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, "uniform-ball", 30_000, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(out[r] is None for r in range(1, world))
    assert np.array_equal(out[0], whole(generate("uniform-ball", 30_000, 0)))


def whole(cols):
    if len(cols) == 2:
        return np.sort(oracle.hull2d(*cols).idx)
    return np.sort(oracle.full_hull3d(*cols)[1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, n, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cols = generate(kind, n, 0)
    b = [(n * r) // world for r in range(world + 1)]
    mine = tuple(torch.from_numpy(np.ascontiguousarray(c[b[rank]:b[rank + 1]])) for c in cols)
    res, info = sharded.hull_sharded(mine, b[rank], Tolerance(), return_info=True, **CPU)
    if rank == 0:
        q.put((np.sort(res.numpy()), info["eps"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n", [("uniform-disk", 200_000), ("unit-square", 100_000),
                                    ("near-circle", 100_000), ("uniform-ball", 50_000),
                                    ("unit-cube", 50_000)])
def test_gloo_world2_matches_whole_input(kind, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, eps = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cols = generate(kind, n, 0)
    assert np.array_equal(got, whole(cols))
    # every rank used the whole input's Tolerance.effective
    spans = [float(c.max() - c.min()) for c in cols]
    assert eps == 1e-12 * float(np.hypot.reduce(spans))


def _layered_cube(n_side=12):
    """3D lattice sorted by z: a slice of one z-layer is coplanar."""
    g = np.arange(n_side, dtype=np.float64)
    z, y, x = np.meshgrid(g, g, g, indexing="ij")
    rng = np.random.default_rng(5)
    jit = lambda a: a + rng.uniform(-1e-3, 1e-3, a.shape) * (a > 0) * (a < n_side - 1)
    return tuple(np.ascontiguousarray(c.ravel()) for c in (jit(x), jit(y), z))


def _worker_cols(rank, world, port, cols, q, fail_rank):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    n = cols[0].size
    b = [(n * r) // world for r in range(world + 1)]
    mine = tuple(torch.from_numpy(np.ascontiguousarray(c[b[rank]:b[rank + 1]])) for c in cols)
    hooks = dict(CPU)
    if rank == fail_rank:
        def boom(*a):
            raise MemoryError("simulated device failure")
        hooks["local_hull"] = boom
    try:
        res = sharded.hull_sharded(mine, b[rank], Tolerance(), **hooks)
        q.put((rank, "ok", None if res is None else np.sort(res.numpy())))
    except RuntimeError as e:
        q.put((rank, "raised", str(e)))
    dist.destroy_process_group()


def _run_world(cols, world, fail_rank=-1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_cols, args=(r, world, port, cols, q, fail_rank)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (st, v)) for r, st, v in (q.get(timeout=240) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_gloo_degenerate_slice_contributes_its_points():
    # 3 ranks over a 12-layer lattice sorted by z: rank 0's slice is
    # layers 0-3, a full 3D set; with 12 ranks each slice would be a plane.
    cols = _layered_cube()
    n = cols[0].size
    world = 12  # one coplanar z-layer per rank
    out = _run_world(cols, world)
    assert out[0][0] == "ok"
    assert np.array_equal(out[0][1], whole(cols))


def test_gloo_failure_raises_on_every_rank():
    cols = generate("uniform-ball", 20_000, 2)
    out = _run_world(cols, 2, fail_rank=1)
    for r in (0, 1):
        st, msg = out[r]
        assert st == "raised" and "rank(s) [1]" in msg


@pytest.mark.parametrize("nshards", [1, 3, 8])
def test_loopback_cpu(nshards):
    for kind, n in (("uniform-disk", 100_000), ("uniform-ball", 30_000)):
        cols = generate(kind, n, 1)
        got = sharded.hull_sharded_loopback(tuple(torch.from_numpy(c) for c in cols), nshards, **CPU)
        assert np.array_equal(np.sort(got.numpy()), whole(cols))


def test_hypot_reduce_matches_numpy():
    rng = np.random.default_rng(1)
    for _ in range(200):
        s = rng.random(3) * 10.0 ** rng.integers(-5, 5)
        assert sharded.hypot_reduce(s) == float(np.hypot.reduce(s))
        assert sharded.hypot_reduce(s[:2]) == float(np.hypot.reduce(s[:2]))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [("uniform-disk", 4_000_000), ("unit-square", 1_000_000),
                                    ("uniform-ball", 2_000_000), ("unit-cube", 2_000_000)])
def test_loopback_gpu_matches_single(kind, n):
    cols = generate(kind, n, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    for p in (2, 8):
        got, info = sharded.hull_sharded_loopback(d, p, return_info=True)
        assert np.array_equal(np.sort(got.cpu().numpy()), whole(cols))
        assert info["union"] >= got.numel()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [("uniform-ball", 2_000_000), ("unit-cube", 1_000_000)])
def test_split_filter_shares_intersect_to_the_hull(kind, n):
    """sh_set_filter_share: every share keeps a superset of the hull, the
    candidates outside the share included; the intersection is the hull."""
    import paper_1201_2936_b200 as P
    cols = generate(kind, n, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    full = P.hull_indices_3d(d)
    for R in (2, 5):
        parts = [P.hull_indices_3d(d, filter_share=(r, R)) for r in range(R)]
        for p in parts:
            assert torch.isin(full, p).all()
        keep = torch.ones(parts[0].numel(), dtype=torch.bool, device=parts[0].device)
        for p in parts[1:]:
            keep &= torch.isin(parts[0], p)
        assert torch.equal(parts[0][keep], full)  # discovery order kept
    assert torch.equal(P.hull_indices_3d(d), full)  # the setting does not persist


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [("uniform-ball", 2_000_000), ("uniform-disk", 2_000_000)])
def test_staged_ranks_emulated_on_one_gpu(kind, n):
    """The product path's two-stage slice hull (sh_hull_shard_begin / _end)
    for two slices in turn, with the statistics of the other slice from
    sh_stats, then the (split) merge: equal to the single hull."""
    cols = generate(kind, n, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    dim = len(cols)
    b = [0, n // 3, n]
    slices = [tuple(c[b[r]:b[r + 1]].contiguous() for c in d) for r in range(2)]
    recs = []
    for r in range(2):
        staged = sharded.StagedDeviceHull()
        st = staged.begin(slices[r], b[r], Tolerance())
        other = sharded.device_stats(slices[1 - r], b[1 - r])
        gstats = sharded.device_reduce_stats(torch.stack([st, other] if r == 0 else [other, st]), dim)
        gidx, coords, eps = staged.end(slices[r], b[r], Tolerance(), gstats)
        recs.append(torch.cat([coords, gidx.to(torch.float64)[:, None]], dim=1))
    union = torch.cat(recs)
    split = [sharded._merge(union, dim, eps, sharded.device_merge_hull, share=(r, 2) if dim == 3 else None)
             for r in range(2)]
    got = split[0][torch.isin(split[0], split[1])]
    assert np.array_equal(np.sort(got.cpu().numpy()), whole(cols))


@pytest.mark.gpu
def test_device_bbox_matches_numpy():
    cols = generate("uniform-ball", 1_000_001, 3)
    bb = sharded.device_bbox(tuple(torch.from_numpy(c).cuda() for c in cols)).cpu().numpy()
    assert np.array_equal(bb, np.array([c.min() for c in cols] + [c.max() for c in cols]))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,offset", [("uniform-disk", 300_001, 0), ("unit-square", 50_000, 7_000_000),
                                           ("uniform-ball", 200_003, 123), ("unit-cube", 1000, 5)])
def test_device_stats_match_host(kind, n, offset):
    cols = generate(kind, n, 4)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    got = sharded.device_stats(d, offset).cpu().numpy()
    assert np.array_equal(got, cpu_stats(tuple(torch.from_numpy(c) for c in cols), offset).numpy())
    # and the reduction over "ranks"
    parts = [sharded.device_stats(tuple(c[a:b] for c in d), offset + a)
             for a, b in ((0, n // 3), (n // 3, n - 10), (n - 10, n))]
    g = sharded.device_reduce_stats(torch.stack(parts), len(cols)).cpu().numpy()
    assert np.array_equal(g, got)


def _nccl_worker(rank, world, port, kind, n, q):
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    cols = generate(kind, n, 0)
    b = [(n * r) // world for r in range(world + 1)]
    mine = tuple(torch.from_numpy(np.ascontiguousarray(c[b[rank]:b[rank + 1]])).cuda() for c in cols)
    res = sharded.hull_sharded(mine, b[rank])
    if rank == 0:
        q.put(np.sort(res.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("kind,n", [("uniform-disk", 2_000_000), ("uniform-ball", 1_000_000)])
def test_nccl_world2_matches_single(kind, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, kind, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cols = generate(kind, n, 0)
    assert np.array_equal(got, whole(cols))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n", [("uniform-disk", 3_000_000), ("uniform-ball", 1_000_000),
                                    ("unit-cube", 200_000), ("near-circle", 500_000)])
def test_nccl_world1_staged_matches_single(kind, n):
    """The product path on a one-rank communicator (the plain hull, no
    exchange): equal to the single hull."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    p = ctx.Process(target=_nccl_worker, args=(0, 1, port, kind, n, q))
    p.start()
    got = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    cols = generate(kind, n, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    import paper_1201_2936_b200 as P
    single = P.hull_indices_2d(d) if len(cols) == 2 else P.hull_indices_3d(d)
    assert np.array_equal(got, np.sort(single.cpu().numpy()))

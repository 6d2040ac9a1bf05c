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
from paper_1201_2936_b200.geometry import Tolerance


def cpu_bbox(cols):
    return torch.tensor([float(c.min()) for c in cols] + [float(c.max()) for c in cols],
                        dtype=torch.float64)


def cpu_hull(cols, tol):
    """Oracle stand-in for the device hull (exact reference semantics)."""
    arrs = [c.numpy() for c in cols]
    if len(arrs) == 2:
        r = oracle.hull2d(*arrs, eps_rel=tol.eps_rel, eps_abs=tol.eps_abs)
        return torch.from_numpy(r.idx.copy())
    _, idx, _ = oracle.full_hull3d(*arrs, eps_rel=tol.eps_rel, eps_abs=tol.eps_abs)
    return torch.from_numpy(np.asarray(idx, dtype=np.int64).copy())


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
    res, info = sharded.hull_sharded(mine, b[rank], Tolerance(), local_hull=cpu_hull,
                                     local_bbox=cpu_bbox, return_info=True)
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


@pytest.mark.parametrize("nshards", [1, 3, 8])
def test_loopback_cpu(nshards):
    for kind, n in (("uniform-disk", 100_000), ("uniform-ball", 30_000)):
        cols = generate(kind, n, 1)
        got = sharded.hull_sharded_loopback(tuple(torch.from_numpy(c) for c in cols), nshards,
                                            local_hull=cpu_hull, local_bbox=cpu_bbox)
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
def test_device_bbox_matches_numpy():
    cols = generate("uniform-ball", 1_000_001, 3)
    bb = sharded.device_bbox(tuple(torch.from_numpy(c).cuda() for c in cols)).cpu().numpy()
    assert np.array_equal(bb, np.array([c.min() for c in cols] + [c.max() for c in cols]))

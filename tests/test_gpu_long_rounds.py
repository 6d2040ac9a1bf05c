"""GPU: the streaming long-segment round kernel (k_stream,
csrc/sh_stream.cuh) on every peeled round, including its point-by-point
path for chunks that overlap three or more segments: the thresholds are
lowered through SH_LONG_MIN_LIVE / SH_LONG_SEG_MIN so that rounds 2-6 of
small and fragmented inputs all take it.  Bar: identical vertex lists
(discovery order in 2D), iterations and per-round traces vs the oracle."""

import os

import numpy as np
import pytest
import torch

import oracle
import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate

pytestmark = pytest.mark.gpu


@pytest.fixture
def force_long(monkeypatch):
    monkeypatch.setenv("SH_LONG_MIN_LIVE", "0")
    monkeypatch.setenv("SH_LONG_SEG_MIN", "1")


@pytest.mark.parametrize("kind,n,seed", [("uniform-disk", 300_000, 1), ("on-circle", 200_000, 2),
                                          ("near-circle", 200_000, 3), ("unit-square", 50_000, 4),
                                          ("on-circle", 3_000, 5), ("on-circle", 600, 6), ("near-circle", 900, 7)])
def test_2d_every_peeled_round_long(force_long, kind, n, seed):
    cols = generate(kind, n, seed)
    idx, res = P.hull_indices_2d(tuple(torch.from_numpy(c).cuda() for c in cols), return_info=True)
    o = oracle.hull2d(*cols)
    assert np.array_equal(idx.cpu().numpy(), o.idx)
    assert res.iterations == o.iterations
    assert np.array_equal(P.trace()[:, :3], o.trace)


@pytest.mark.parametrize("kind,n,seed", [("uniform-ball", 200_000, 1), ("on-sphere", 20_000, 2), ("on-sphere", 500, 5),
                                          ("near-sphere", 100_000, 3), ("unit-cube", 100_000, 4)])
def test_3d_every_peeled_round_long(force_long, kind, n, seed):
    cols = generate(kind, n, seed)
    idx, _, res = P.hull_indices_3d(tuple(torch.from_numpy(c).cuda() for c in cols), return_info=True)
    o, ref, _ = oracle.full_hull3d(*cols)
    assert res.iterations == o.iterations and res.candidates == len(o.idx)
    assert np.array_equal(np.sort(idx.cpu().numpy()), np.sort(ref))
    tr = P.trace()
    assert np.array_equal(tr[:, :3], o.trace)


def test_default_thresholds_restored():
    assert "SH_LONG_MIN_LIVE" not in os.environ
    cols = generate("uniform-disk", 100_000, 7)
    idx = P.hull_indices_2d(tuple(torch.from_numpy(c).cuda() for c in cols)).cpu().numpy()
    assert np.array_equal(idx, oracle.hull2d(*cols).idx)

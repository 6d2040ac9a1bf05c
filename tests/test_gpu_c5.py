"""GPU, full size: BASELINE config C5 -- 3D Quickhull of 200M points uniform
in the ball (seed 0), the north star's sharded configuration.

Single GPU: the device loop equals the oracle's restatement of the
reference loop (candidate set in discovery order, rounds, per-round trace)
and the final vertex set equals Qhull on the candidates (the reference's own
filter is infeasible at this size).  Sharded, in loopback
(P slices hulled one after the other on this GPU, the merge on the union):
P = 2, 4, 8 give the single-GPU vertex set.  About 3 minutes, most of it the
host generator and the oracle loop."""

import numpy as np
import pytest
import torch

import oracle
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import sharded
from paper_1201_2936_b200.datagen import generate

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 200_000_000


@pytest.fixture(scope="module")
def c5():
    cols = generate("uniform-ball", N, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    idx, _, res = P.hull_indices_3d(d, return_info=True)
    torch.cuda.synchronize()
    return cols, d, np.sort(idx.cpu().numpy()), res, P.trace()


def test_c5_single_gpu_vs_oracle_and_qhull(c5):
    cols, _, got, res, tr = c5
    o = oracle.hull3d(*cols)
    assert o.status == oracle.STATUS_OK
    assert res.candidates == len(o.idx) and res.iterations == o.iterations
    assert np.array_equal(tr[:, :3], o.trace)
    from scipy.spatial import ConvexHull
    rows = np.column_stack([c[o.idx] for c in cols])
    want = np.sort(o.idx[ConvexHull(rows).vertices])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("nshards", [2, 4, 8])
def test_c5_loopback_equals_single(c5, nshards):
    _, d, got, _, _ = c5
    g, info = sharded.hull_sharded_loopback(d, nshards, return_info=True)
    assert np.array_equal(np.sort(g.cpu().numpy()), got)
    assert info["union"] >= g.numel()

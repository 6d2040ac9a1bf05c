"""GPU: PTS1 files straight into HBM and device-side uniform-box clouds
(SURVEY.md §8(f) rank 4), bit-identical to the host paths."""

import os

import numpy as np
import pytest
import torch

import oracle
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import pointio
from paper_1201_2936_b200.datagen import generate

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name,kind,n,seed", [("sample2d.pts", "uniform-disk", 1000, 5),
                                               ("sample3d.pts", "uniform-ball", 700, 6)])
def test_reference_files_to_device(name, kind, n, seed):
    t = pointio.read_points_binary_device(os.path.join(GOLD, name))
    assert t.is_cuda and t.dtype == torch.float64 and t.shape == (n, len(generate(kind, 1, 0)))
    cols = generate(kind, n, seed)
    assert np.array_equal(t.cpu().numpy(), np.column_stack(cols))
    # the (n, dim) tensor goes to the hull entry points as is
    f = P.hull_indices_2d if t.shape[1] == 2 else P.hull_indices_3d
    a = f(t).cpu().numpy()
    b = f(tuple(torch.from_numpy(c).cuda() for c in cols)).cpu().numpy()
    assert np.array_equal(a, b)


def test_large_file_multi_chunk(tmp_path):
    cols = generate("uniform-disk", 6_000_000, 9)  # 96 MB: two pinned chunks
    p = tmp_path / "big.pts"
    pointio.write_points_binary(p, cols)
    t = pointio.read_points_device(p)
    assert np.array_equal(t.cpu().numpy(), np.column_stack(cols))
    idx = P.hull_indices_2d(t).cpu().numpy()
    o = oracle.hull2d(*cols)
    assert np.array_equal(idx, o.idx)


def test_csv_to_device():
    t = pointio.read_points_device(os.path.join(GOLD, "sample3d.csv"))
    assert np.array_equal(t.cpu().numpy(), np.column_stack(generate("on-sphere", 50, 7)))


def test_empty_file(tmp_path):
    p = tmp_path / "e.pts"
    pointio.write_points_binary(p, np.empty((0, 3)))
    t = pointio.read_points_binary_device(p)
    assert t.shape == (0, 3)


@pytest.mark.parametrize("kind", ["unit-square", "unit-cube"])
@pytest.mark.parametrize("n,seed,start", [(1, 0, 0), (1000, 3, 0), (123_457, 11, 5_000_000),
                                          (2_000_000, 0, 0)])
def test_device_generation_bit_exact(kind, n, seed, start):
    host = generate(kind, n, seed, start=start)
    dev = pointio.generate_device(kind, n, seed, start=start)
    for a, b in zip(dev, host):
        assert np.array_equal(a.cpu().numpy(), b)
    rows = pointio.generate_device(kind, n, seed, start=start, layout="rows")
    assert np.array_equal(rows.cpu().numpy(), np.column_stack(host))


def test_c1_from_device_generation():
    # C1: 1M uniform points in the unit square, generated in HBM
    cols = pointio.generate_device("unit-square", 1_000_000, 0)
    idx, res = P.hull_indices_2d(cols, return_info=True)
    o = oracle.hull2d(*generate("unit-square", 1_000_000, 0))
    assert np.array_equal(idx.cpu().numpy(), o.idx) and res.iterations == o.iterations

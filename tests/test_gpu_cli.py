"""GPU: the CLI's hull and bench commands (reference cli.py:61-83,125-162,
test_cli.py:16-26,59-92,105-118) on the device path."""

import csv
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1201_2936_b200 import cli, pointio
from paper_1201_2936_b200.datagen import generate

pytestmark = pytest.mark.gpu


def test_gen_hull_binary_round_trip(tmp_path, capsys):
    p, o = tmp_path / "d.pts", tmp_path / "h.pts"
    assert cli.main(["gen", "--dist", "uniform-disk", "--n", "20000", "--seed", "1", "--dim", "2", "-o", str(p)]) == 0
    assert cli.main(["hull", str(p), "-o", str(o), "--stats"]) == 0
    out = capsys.readouterr().out
    x, y = generate("uniform-disk", 20000, 1)
    want = oracle.hull2d(x, y)
    assert f"n=20000 hull={len(want.idx)} iterations={want.iterations} ms=" in out
    got = pointio.read_points_device(o).cpu().numpy()
    assert set(map(tuple, got.tolist())) == set(zip(x[want.idx].tolist(), y[want.idx].tolist()))
    # boundary order: counter-clockwise, starting at the lexicographic minimum
    assert tuple(got[0]) == min(map(tuple, got.tolist()))
    a, b = np.roll(got, -1, 0) - got, np.roll(got, -2, 0) - np.roll(got, -1, 0)
    cr = a[:, 0] * b[:, 1] - a[:, 1] * b[:, 0]
    assert np.all(cr > 0)


def test_hull_stdout_csv_3d(tmp_path, capsys):
    p = tmp_path / "b.csv"
    assert cli.main(["gen", "--dist", "uniform-ball", "--n", "3000", "--seed", "2", "--dim", "3", "-o", str(p)]) == 0
    assert cli.main(["hull", str(p)]) == 0
    rows = [tuple(map(float, l.split(","))) for l in capsys.readouterr().out.strip().splitlines()]
    x, y, z = generate("uniform-ball", 3000, 2)
    _, ref, _ = oracle.full_hull3d(x, y, z)
    assert set(rows) == set(zip(x[ref].tolist(), y[ref].tolist(), z[ref].tolist()))


def test_hull_degenerate_exit_code(tmp_path):
    p = tmp_path / "flat.pts"
    pointio.write_points_binary(p, np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0.0]]))
    assert cli.main(["hull", str(p)]) == 1


def test_bench_csv(tmp_path):
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--dists", "unit-square,uniform-disk", "--sizes", "1000,50000", "--reps", "2",
                     "--dim", "2", "-o", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert tuple(rows[0]) == cli.BENCH_HEADER
    assert len(rows) == 1 + 2 * 2 * 2
    for r in rows[1:]:
        kind, n, dim, seed = r[0], int(r[1]), int(r[2]), int(r[3])
        assert float(r[4]) > 0
        o = oracle.hull2d(*generate(kind, n, seed))
        assert int(r[5]) == o.iterations and int(r[6]) == len(o.idx)


def test_module_entry_point(tmp_path):
    p = tmp_path / "c.pts"
    r = subprocess.run([sys.executable, "-m", "paper_1201_2936_b200", "gen", "--dist", "unit-cube", "--n", "500",
                        "--seed", "0", "--dim", "3", "-o", str(p)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([sys.executable, "-m", "paper_1201_2936_b200", "hull", str(p), "--stats"],
                       capture_output=True, text=True)
    assert r.returncode == 0 and "n=500 hull=" in r.stdout, r.stderr

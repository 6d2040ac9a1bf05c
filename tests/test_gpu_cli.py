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


GOLD = None


def _gold():
    global GOLD
    if GOLD is None:
        import json
        import os
        GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                           "golden_checks.json")))
    return GOLD


def test_device_giftwrap_matches_reference():
    """sh_giftwrap_2d against the reference's hull2_giftwrap outputs (same
    vertices, same CCW order from the lexicographic minimum), and against
    the sequential oracle on larger clouds."""
    import torch
    from oracle import checks
    from paper_1201_2936_b200.quickhull import giftwrap_2d
    for case in _gold():
        if case["dim"] != 2:
            continue
        rows = np.array(case["rows"])
        idx = giftwrap_2d(torch.tensor(rows, device="cuda"), case["eps"]).cpu().numpy()
        assert rows[idx].tolist() == case["hull"], case["name"]
    for kind, n, seed in (("uniform-disk", 20000, 3), ("on-circle", 1000, 1), ("unit-square", 50000, 2)):
        x, y = generate(kind, n, seed)
        eps = 1e-12 * float(np.hypot(x.max() - x.min(), y.max() - y.min()))
        got = giftwrap_2d(torch.tensor(np.stack([x, y], 1), device="cuda"), eps).cpu().numpy()
        want = checks.giftwrap2d(x, y, eps) if n <= 20000 else None
        if want is not None:
            assert got.tolist() == want
        o = oracle.hull2d(x, y)
        assert set(zip(x[got].tolist(), y[got].tolist())) == set(zip(x[o.idx].tolist(), y[o.idx].tolist()))


def test_device_giftwrap_ties_duplicates_offsets():
    """Adversarial ties: duplicated points, a tiny circle far from the
    origin (differences round to equal values), collinear grids; the
    device walk visits the same coordinates as the sequential C scan."""
    import torch
    from paper_1201_2936_b200.quickhull import giftwrap_2d
    rng = np.random.default_rng(11)
    x, y = generate("on-circle", 6000, 3)
    d = rng.integers(0, 6000, 1500)
    cases = [(np.concatenate([x, x[d]]), np.concatenate([y, y[d]]))]
    cases.append((x * 1e-7 + 1e3, y * 1e-7 - 2e3))
    g = np.arange(40.0)
    X, Y = np.meshgrid(g, g)
    cases.append((X.ravel() * 0.1, Y.ravel() * 0.3))
    for cx, cy in cases:
        eps = 1e-12 * float(np.hypot(cx.max() - cx.min(), cy.max() - cy.min()))
        got = giftwrap_2d(torch.tensor(np.stack([cx, cy], 1), device="cuda"), eps).cpu().numpy()
        want = oracle.giftwrap2d(cx, cy, eps)
        assert np.array_equal(cx[got], cx[want]) and np.array_equal(cy[got], cy[want])


def test_device_giftwrap_dense_circle_digest():
    """Sequential-scan semantics where ties within eps abound: the device
    walk equals the C restatement of hull2_giftwrap index for index."""
    import hashlib
    import json
    import os
    import torch
    from paper_1201_2936_b200.quickhull import giftwrap_2d
    for g in json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                         "golden_checks_big.json"))):
        x, y = generate(g["kind"], g["n"], g["seed"])
        idx = giftwrap_2d(torch.tensor(np.stack([x, y], 1), device="cuda"), g["eps"]).cpu().numpy()
        assert idx.size == g["h"]
        assert hashlib.sha256(idx.astype("<i8").tobytes()).hexdigest() == g["sha256"]


def test_verify_2d_and_3d(tmp_path, capsys):
    src = tmp_path / "d.csv"
    assert cli.main(["gen", "--dist", "uniform-disk", "--n", "200", "--seed", "5", "--dim", "2", "-o", str(src)]) == 0
    assert cli.main(["verify", str(src)]) == 0
    assert capsys.readouterr().out.strip().endswith("hull vertices match the oracle")
    big = tmp_path / "big.pts"
    assert cli.main(["gen", "--dist", "uniform-disk", "--n", "1000000", "--seed", "1", "--dim", "2", "-o", str(big)]) == 0
    assert cli.main(["verify", str(big)]) == 0
    assert "hull vertices match the oracle" in capsys.readouterr().out
    # dense circle: the gift wrap and Quickhull resolve within-eps ties
    # differently, so the reference's own verify reports a mismatch here
    # (counts from the sequential C restatement, golden_checks_big.json)
    circ = tmp_path / "circ.pts"
    assert cli.main(["gen", "--dist", "on-circle", "--n", "100000", "--seed", "1", "--dim", "2", "-o", str(circ)]) == 0
    assert cli.main(["verify", str(circ)]) == 1
    assert "MISMATCH: 214 oracle vertices missing, 124 unexpected" in capsys.readouterr().err
    small = tmp_path / "ball.csv"
    assert cli.main(["gen", "--dist", "uniform-ball", "--n", "48", "--seed", "9", "--dim", "3", "-o", str(small)]) == 0
    assert cli.main(["verify", str(small)]) == 0
    assert "ok: oracle vertices covered; extras=0" in capsys.readouterr().out
    big3 = tmp_path / "big3.csv"
    assert cli.main(["gen", "--dist", "uniform-ball", "--n", "200", "--seed", "9", "--dim", "3", "-o", str(big3)]) == 0
    assert cli.main(["verify", str(big3)]) == 2
    assert "3D verification is capped at n=128" in capsys.readouterr().err


def test_verify_pipeline_20_seeds(tmp_path):
    """Acceptance criterion 8 (reference test_acceptance.py:175-197)."""
    for seed in range(20):
        src, out = str(tmp_path / f"d{seed}.csv"), str(tmp_path / f"h{seed}.csv")
        codes = (cli.main(["gen", "--dist", "uniform-disk", "--n", "256", "--seed", str(seed), "--dim", "2", "-o", src]),
                 cli.main(["hull", src, "-o", out]), cli.main(["verify", src]))
        assert codes == (0, 0, 0), (seed, codes)


def test_bench_plot_and_threads(tmp_path, capsys):
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--dists", "uniform-disk,on-circle", "--sizes", "128,1024", "--reps", "3", "--dim", "2",
                     "-o", str(out), "--plot", "--threads", "2"]) == 0
    fig = tmp_path / ("bench.png" if cli._have_matplotlib() else "bench.svg")
    assert fig.stat().st_size > 0
    assert str(fig) in capsys.readouterr().out
    rows = list(csv.reader(open(out)))[1:]
    iters = {(r[0], int(r[1])): int(r[5]) for r in rows}
    assert iters[("on-circle", 1024)] > iters[("uniform-disk", 1024)]
    src = tmp_path / "c.csv"
    assert cli.main(["gen", "--dist", "on-circle", "--n", "12", "--seed", "2", "--dim", "2", "-o", str(src)]) == 0
    assert cli.main(["hull", str(src), "--stats", "--threads", "2"]) == 0
    assert "hull=12" in capsys.readouterr().out

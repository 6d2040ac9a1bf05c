"""CPU: the CLI's argument handling, usage errors and exit codes (reference
cli.py:165-233, test_cli.py:28-45,120-128) and `gen` output; the GPU
commands are covered by tests/test_gpu_cli.py."""

import os

import numpy as np

from paper_1201_2936_b200 import cli, pointio
from paper_1201_2936_b200.datagen import generate


def test_gen_writes_reference_formats(tmp_path):
    p = tmp_path / "d.pts"
    assert cli.main(["gen", "--dist", "uniform-disk", "--n", "1000", "--seed", "5", "--dim", "2", "-o", str(p)]) == 0
    assert p.read_bytes() == open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sample2d.pts"), "rb").read()
    c = tmp_path / "s.csv"
    assert cli.main(["gen", "--dist", "on-sphere", "--n", "50", "--seed", "7", "--dim", "3", "-o", str(c)]) == 0
    ps = pointio.read_points_csv(c)
    assert all(np.array_equal(a, b) for a, b in zip(ps.coords, generate("on-sphere", 50, 7)))


def test_usage_errors(tmp_path):
    out = str(tmp_path / "x.pts")
    assert cli.main(["gen", "--dist", "uniform-disk", "--n", "10", "--seed", "0", "--dim", "3", "-o", out]) == 2
    assert cli.main(["gen", "--dist", "nope", "--n", "10", "--seed", "0", "--dim", "2", "-o", out]) == 2
    # Distribution's band check (reference datagen.py:45-46 -> exit code 2)
    assert cli.main(["gen", "--dist", "near-circle", "--n", "10", "--seed", "0", "--dim", "2", "--band", "1.5",
                     "-o", out]) == 2
    assert not os.path.exists(out)
    assert cli.main(["bench", "--dists", "", "--sizes", "10", "--dim", "2", "-o", out]) == 2
    assert cli.main(["bench", "--dists", "uniform-ball", "--sizes", "10", "--dim", "2", "-o", out]) == 2
    assert cli.main(["bench", "--dists", "uniform-disk", "--sizes", "0", "--dim", "2", "-o", out]) == 2
    assert cli.main(["bench", "--dists", "uniform-disk", "--sizes", "x", "--dim", "2", "-o", out]) == 2
    assert cli.main(["bench", "--dists", "uniform-disk", "--sizes", "10", "--reps", "0", "--dim", "2", "-o", out]) == 2
    assert cli.main([]) == 2


def test_unwritable_and_bad_input(tmp_path):
    assert cli.main(["gen", "--dist", "uniform-disk", "--n", "10", "--seed", "0", "--dim", "2",
                     "-o", str(tmp_path / "no" / "x.pts")]) == 1
    bad = tmp_path / "bad.pts"
    bad.write_bytes(b"PTS1\x09\x00")
    assert cli.main(["hull", str(bad)]) == 1

"""CPU: the brute-force checks behind the CLI's `verify` (reference
oracle.py:20-52,82-118) -- the oracle restatement and the CLI's numpy 3D
check against golden vectors from the reference's own oracles
(tests/golden/make_golden_checks.py)."""

import json
import os

import numpy as np
import pytest

from oracle import checks
from paper_1201_2936_b200 import cli
from paper_1201_2936_b200.errors import ContractViolation, DegenerateInputError

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_checks.json")))


@pytest.mark.parametrize("case", [c for c in GOLD if c["dim"] == 2], ids=lambda c: c["name"])
def test_giftwrap_oracle_matches_reference(case):
    rows = np.array(case["rows"])
    idx = checks.giftwrap2d(rows[:, 0], rows[:, 1], case["eps"])
    assert rows[idx].tolist() == case["hull"]


@pytest.mark.parametrize("case", [c for c in GOLD if c["dim"] == 3], ids=lambda c: c["name"])
def test_bruteforce3d_matches_reference(case):
    rows = np.array(case["rows"])
    want = set(map(tuple, case["hull"]))
    assert set(map(tuple, rows[checks.bruteforce3d(rows, case["eps"])].tolist())) == want
    # the CLI's vectorised check (product code, no GPU needed)
    assert cli._support_planes_3d(rows, case["eps"]) == want


def test_3d_extras_within_eps():
    case = next(c for c in GOLD if c["name"] == "uniform-ball")
    rows = np.array(case["rows"])
    eps = case["eps"]
    c = rows.mean(axis=0)
    assert not cli._near_or_outside_3d(rows, c, eps)  # deep interior
    assert cli._near_or_outside_3d(rows, c + 10.0, eps)  # outside
    v = np.array(case["hull"][0])
    assert cli._near_or_outside_3d(rows, v, eps)  # on the boundary


def test_3d_check_errors():
    with pytest.raises(ContractViolation):
        cli._support_planes_3d(np.zeros((3, 3)), 0.0)
    flat = np.array([[0, 0, 1], [1, 0, 1], [0, 1, 1], [1, 1, 1], [0.3, 0.4, 1.0]])
    with pytest.raises(DegenerateInputError):
        cli._support_planes_3d(flat, 1e-12)


def test_verify_parser_surface():
    p = cli._build_parser()
    a = p.parse_args(["verify", "x.pts", "--eps-rel", "1e-9"])
    assert a.func is cli.cmd_verify and a.eps_rel == 1e-9
    assert p.parse_args(["hull", "x.pts", "--threads", "2"]).threads == 2
    b = p.parse_args(["bench", "--dists", "uniform-disk", "--sizes", "8", "--dim", "2", "-o", "b.csv", "--plot"])
    assert b.plot == "" and b.threads is None
    assert p.parse_args(["bench", "--dists", "uniform-disk", "--sizes", "8", "--dim", "2", "-o", "b.csv",
                         "--plot", "f.svg"]).plot == "f.svg"


def test_bench_figure_svg(tmp_path):
    rows = [("uniform-disk", 128, 2, 0, "0.5", 3, 10), ("uniform-disk", 1024, 2, 0, "0.7", 5, 14),
            ("on-circle", 128, 2, 0, "0.6", 8, 128), ("on-circle", 1024, 2, 1, "1.2", 11, 1024)]
    f = tmp_path / "b.svg"
    cli._render_bench_figure(str(f), rows)
    assert f.stat().st_size > 0
    if not cli._have_matplotlib():
        txt = f.read_text()
        assert txt.startswith("<svg") and txt.count("<polyline") == 4 and "on-circle" in txt


@pytest.mark.parametrize("case", [c for c in GOLD if c["dim"] == 2], ids=lambda c: c["name"])
def test_giftwrap_c_oracle_matches_reference(case):
    import oracle
    rows = np.array(case["rows"])
    idx = oracle.giftwrap2d(rows[:, 0], rows[:, 1], case["eps"])
    assert rows[idx].tolist() == case["hull"]
    assert idx.tolist() == checks.giftwrap2d(rows[:, 0], rows[:, 1], case["eps"])

"""CPU: the PTS1 / CSV readers' validation and parsing against the
reference's own files and error messages (pointfile.py:37-118).  The device
transfer itself is covered by tests/test_gpu_pointio.py."""

import os
import struct
import sys

import numpy as np
import pytest

from paper_1201_2936_b200 import pointio
from paper_1201_2936_b200.datagen import generate

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REF = "/root/reference/pkg/src"
HAVE_REF = os.path.isdir(REF)


def ref_pointfile():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from seghull import pointfile
    return pointfile


@pytest.mark.parametrize("name,dim,n", [("sample2d.pts", 2, 1000), ("sample3d.pts", 3, 700)])
def test_header_of_reference_files(name, dim, n):
    assert pointio.read_header(os.path.join(GOLD, name)) == (dim, n)


def test_reference_payload_is_the_generator_cloud():
    blob = open(os.path.join(GOLD, "sample2d.pts"), "rb").read()
    rows = np.frombuffer(blob, "<f8", offset=16).reshape(-1, 2)
    x, y = generate("uniform-disk", 1000, 5)
    assert np.array_equal(rows[:, 0], x) and np.array_equal(rows[:, 1], y)


def bad_files(tmp_path):
    good = struct.pack("<4sIQ", b"PTS1", 2, 3) + np.arange(6, dtype="<f8").tobytes()
    cases = {
        "truncated": b"PTS1\x02",
        "magic": b"PTS2" + good[4:],
        "dim": struct.pack("<4sIQ", b"PTS1", 4, 1) + bytes(32),
        "size": good[:-8],
    }
    out = {}
    for k, blob in cases.items():
        p = tmp_path / f"{k}.pts"
        p.write_bytes(blob)
        out[k] = p
    return out


def test_header_errors(tmp_path):
    files = bad_files(tmp_path)
    for k, p in files.items():
        with pytest.raises(pointio.PointFileError):
            pointio.read_header(p)
    with pytest.raises(pointio.PointFileError):
        pointio.read_header(tmp_path / "missing.pts")


@pytest.mark.skipif(not HAVE_REF, reason="reference not present (GPU box)")
def test_header_error_messages_match_reference(tmp_path):
    pf = ref_pointfile()
    for k, p in bad_files(tmp_path).items():
        with pytest.raises(pf.PointFileError) as want:
            pf.read_points_binary(p)
        with pytest.raises(pointio.PointFileError) as got:
            pointio.read_header(p)
        assert str(got.value) == str(want.value), k


def test_csv_reader_matches_golden(tmp_path):
    ps = pointio.read_points_csv(os.path.join(GOLD, "sample3d.csv"))
    assert ps.dim == 3 and ps.n == 50
    from paper_1201_2936_b200.datagen import generate as g
    cols = g("on-sphere", 50, 7)
    for a, b in zip(ps.coords, cols):
        assert np.array_equal(a, b)  # repr() round-trips every double


@pytest.mark.skipif(not HAVE_REF, reason="reference not present (GPU box)")
def test_csv_errors_match_reference(tmp_path):
    pf = ref_pointfile()
    cases = {"cols": "1,2,3,4\n", "incons": "1,2\n1,2,3\n", "comment": "1,2\n# x\n", "nan": "1,zz\n",
             "empty": "\n\n"}
    for k, txt in cases.items():
        p = tmp_path / f"{k}.csv"
        p.write_text(txt)
        with pytest.raises(pf.PointFileError) as want:
            pf.read_points_csv(p)
        with pytest.raises(pointio.PointFileError) as got:
            pointio.read_points_csv(p)
        assert str(got.value) == str(want.value), k
    p = tmp_path / "hdr.csv"
    p.write_text("# x,y,z\n")
    assert pointio.read_points_csv(p).dim == 3


def test_writer_matches_reference_bytes(tmp_path):
    x, y, z = generate("uniform-ball", 700, 6)
    p = tmp_path / "w.pts"
    pointio.write_points_binary(p, (x, y, z))
    assert p.read_bytes() == open(os.path.join(GOLD, "sample3d.pts"), "rb").read()


def test_device_generation_rejects_libm_kinds():
    with pytest.raises(ValueError):
        pointio.generate_device("uniform-disk", 10)

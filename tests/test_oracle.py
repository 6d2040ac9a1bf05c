"""The oracle (oracle/qh_oracle.c, a plain-C restatement of the reference
drivers) pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle
from golden_io import load, rows_of

CASES = load()
C2 = [c for c in CASES if c.dim == 2]
C3 = [c for c in CASES if c.dim == 3]


@pytest.mark.parametrize("case", C2, ids=[c.name for c in C2])
def test_oracle_2d_matches_reference(case):
    r = oracle.hull2d(*case.coords)
    # quickhull_2d never raises for n > 0
    assert case.error is None and r.status == oracle.STATUS_OK
    got = rows_of(case.coords, r.idx)
    # vertices byte-identical, in the reference's discovery order
    assert got.tobytes() == case.verts.tobytes()
    assert r.iterations == case.iterations
    assert case.n - len(r.idx) == case.discarded
    assert oracle.warnings_2d(r, case.n) == case.warnings
    assert r.trace.tolist() == case.trace


# reference cases (tests/golden/make_golden.py degenerate_3d) whose loop
# candidates include points on the hull's faces or edges
DEGENERATE_FILTER = {"lattice-cube-3", "lattice-cube-4", "lattice-cube-5", "lattice-cube-7",
                     "cube-faces-300", "cube-faces-1500", "rings-120"}


@pytest.mark.parametrize("case", C3, ids=[c.name for c in C3])
def test_oracle_3d_matches_reference(case):
    r = oracle.hull3d(*case.coords)
    if case.error:
        assert case.error == "DegenerateInputError" and r.status == oracle.STATUS_DEGENERATE
        return
    assert r.status == oracle.STATUS_OK
    assert r.iterations == case.iterations
    assert r.trace.tolist() == case.trace
    if case.cand is not None:
        # loop candidates identical and in order (input of _extreme_vertex_mask)
        assert rows_of(case.coords, r.idx).tobytes() == case.cand.tobytes()
    if case.name in DEGENERATE_FILTER:
        # coplanar / collinear candidates: the reference's eps-tolerant filter
        # keeps boundary points that Qhull's strict extreme set drops; the
        # oracle pins the loop only, the GPU test pins the filter against
        # these reference outputs (tests/test_gpu_parity.py::test_golden_3d)
        keep = oracle.extreme_filter_qhull(case.cand)
        assert np.all(case.keep[keep])  # every strict vertex is kept by the reference
        return
    if case.cand is not None:
        # the exact extreme-point set equals the reference's filter result
        keep = oracle.extreme_filter_qhull(case.cand)
        assert np.array_equal(keep, case.keep)
    _, idx, warns = oracle.full_hull3d(*case.coords)
    assert rows_of(case.coords, idx).tobytes() == case.verts.tobytes()
    assert warns == case.warnings
    assert case.n - len(idx) == case.discarded


def test_golden_covers_reference_kats():
    names = {c.name for c in CASES}
    for k in ("kat-square-centre", "kat-collinear-2d", "kat-duplicates-2d", "kat-on-edge-2d",
              "kat-cube-centroid", "kat-coplanar-3d", "kat-collinear-3d", "on-circle-1024-s7",
              "on-sphere-512-s3"):
        assert k in names
    circ = next(c for c in CASES if c.name == "on-circle-1024-s7")
    assert circ.h == 1024  # test_quickhull.py:27-31


def test_oracle_empty_input():
    e = np.empty(0)
    assert oracle.hull2d(e, e).status == oracle.STATUS_EMPTY
    assert oracle.hull3d(e, e, e).status == oracle.STATUS_EMPTY

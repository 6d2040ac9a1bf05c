"""GPU: 3D facet output (north star: "facet index triples out"; SURVEY.md
§8(f) rank 3).  The reference returns vertex sets only, so the facets are
pinned to Qhull's simplices on general-position inputs and, everywhere
(including the reference's degenerate KATs: cube + centroid, coincident and
lattice points), to the structural definition of a hull triangulation
(tests/facet_check.py): closed, consistently oriented, Euler, supporting
planes checked exactly, vertices = the returned hull vertices."""

import numpy as np
import pytest
import torch

import paper_1201_2936_b200 as P
from facet_check import canonical, check_mesh, check_supporting, qhull_simplices
from golden_io import load
from paper_1201_2936_b200.datagen import generate

pytestmark = pytest.mark.gpu

C3 = [c for c in load() if c.dim == 3 and not c.error]


def dev(cols):
    return tuple(torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols)


def run(cols, tol=P.Tolerance()):
    idx, fac, res = P.hull_indices_3d(dev(cols), tol, facets=True, return_info=True)
    return idx.cpu().numpy(), fac.cpu().numpy(), res


@pytest.mark.parametrize("case", C3, ids=[c.name for c in C3])
def test_golden_cases_facets(case):
    rows = np.column_stack(case.coords)
    idx, fac, res = run(case.coords)
    assert res.facets == len(fac)
    if len(idx) < 4:
        assert len(fac) == 0  # no 3D hull (single, coincident, collinear, triangle, ...)
        return
    v = check_mesh(fac)
    assert set(v.tolist()) <= set(idx.tolist())
    check_supporting(rows, fac)
    if case.name.startswith(("uniform-ball", "on-sphere", "near-sphere", "unit-cube")):
        assert set(v.tolist()) == set(idx.tolist())
        assert canonical(fac) == canonical(qhull_simplices(rows))


@pytest.mark.parametrize("kind", ["uniform-ball", "unit-cube", "on-sphere", "near-sphere"])
@pytest.mark.parametrize("n", [5_000, 200_000])
def test_random_clouds_equal_qhull(kind, n):
    cols = generate(kind, n, 3)
    rows = np.column_stack(cols)
    idx, fac, res = run(cols)
    v = check_mesh(fac)
    assert set(v.tolist()) == set(idx.tolist())
    assert canonical(fac) == canonical(idx[qhull_simplices(rows[idx])])
    check_supporting(rows[idx], _local(idx, fac), exact=False)


def _local(idx, fac):
    order = np.argsort(idx)
    pos = np.empty(idx.max() + 1, np.int64)
    pos[idx[order]] = order
    return pos[fac]


def test_cube_corners_and_lattice_are_triangulated():
    # 8 cube corners + centre: 6 coplanar quads -> 12 triangles
    g = np.array([[x, y, z] for x in (0.0, 1.0) for y in (0.0, 1.0) for z in (0.0, 1.0)] + [[0.5, 0.5, 0.5]])
    idx, fac, _ = run(tuple(g.T.copy()))
    assert len(fac) == 12
    check_mesh(fac)
    check_supporting(g, fac, exact=True)
    # integer lattice 6^3 (plus duplicates): every hull face has many coplanar points
    L = np.array([[x, y, z] for x in range(6) for y in range(6) for z in range(6)], dtype=np.float64)
    L = np.concatenate([L, L[::7]])
    idx, fac, _ = run(tuple(L.T.copy()))
    v = check_mesh(fac)
    assert set(v.tolist()) <= set(idx.tolist())
    check_supporting(L, fac, exact=True)


def test_ball_1m_and_facet_count():
    cols = generate("uniform-ball", 1_000_000, 0)
    rows = np.column_stack(cols)
    idx, fac, res = run(cols)
    v = check_mesh(fac)
    assert set(v.tolist()) == set(idx.tolist())
    assert len(fac) == 2 * len(idx) - 4
    assert canonical(fac) == canonical(idx[qhull_simplices(rows[idx])])


def test_facets_with_vertices_only_graph_interleaved():
    cols = generate("uniform-ball", 100_000, 1)
    a = P.hull_indices_3d(dev(cols))
    i2, f2 = P.hull_indices_3d(dev(cols), facets=True)
    b = P.hull_indices_3d(dev(cols))
    assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())
    assert np.array_equal(a.cpu().numpy(), i2.cpu().numpy())
    check_mesh(f2.cpu().numpy())


def test_quickhull_3d_facets_field():
    cols = generate("unit-cube", 20_000, 2)
    r = P.quickhull_3d(P.PointSet(cols), facets=True)
    assert r.facets is not None and r.facets.shape == (2 * r.vertices.n - 4, 3)
    assert set(np.unique(r.facets).tolist()) == set(r.indices.tolist())


def test_facet_capacity_retry_surface_cloud():
    # every point is a vertex: the shim's first facet buffer is too small
    cols = generate("on-sphere", 50_000, 4)
    idx, fac, res = run(cols)
    assert len(idx) == 50_000 and len(fac) == 2 * 50_000 - 4
    check_mesh(fac)


def test_small_facet_cap_is_a_contract_error():
    cols = generate("uniform-ball", 10_000, 0)
    d = dev(cols)
    import ctypes
    from paper_1201_2936_b200 import _lib
    out = torch.empty(10_000, dtype=torch.int64, device="cuda")
    fout = torch.empty((10, 3), dtype=torch.int32, device="cuda")
    res = _lib.ShResult()
    rc = _lib.lib().sh_hull3d(_lib.context(0), d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), 1, 10_000,
                              1e-12, float("nan"), out.data_ptr(), fout.data_ptr(), 10, ctypes.byref(res),
                              torch.cuda.current_stream().cuda_stream)
    assert rc == _lib.SH_CONTRACT and res.facets > 10
    assert "facet_cap" in _lib.last_error()


def test_large_degenerate_grids():
    # a 16^3 lattice and a 24 x 24 grid on each face of a cube: hull faces
    # with hundreds of coplanar vertices, triangulated consistently by SoS
    g = np.arange(16, dtype=np.float64)
    L = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    t = np.linspace(0.0, 1.0, 24)
    u, v = [a.ravel() for a in np.meshgrid(t, t, indexing="ij")]
    faces = []
    for axis in range(3):
        for side in (0.0, 1.0):
            f = np.empty((u.size, 3))
            f[:, axis] = side
            f[:, (axis + 1) % 3] = u
            f[:, (axis + 2) % 3] = v
            faces.append(f)
    S = np.unique(np.concatenate(faces), axis=0)
    for pts in (L, S):
        idx, fac, _ = run(tuple(np.ascontiguousarray(pts.T)))
        vset = check_mesh(fac)
        assert set(vset.tolist()) <= set(idx.tolist())
        check_supporting(pts, fac, exact=False)
        # every facet's corners are coplanar with a face of the box: exact
        # zero-volume checks are in check_supporting; the triangulated area
        # must equal the box's surface area
        a, b, c = pts[fac[:, 0]], pts[fac[:, 1]], pts[fac[:, 2]]
        area = 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=1).sum()
        span = pts.max(0) - pts.min(0)
        want = 2 * (span[0] * span[1] + span[1] * span[2] + span[0] * span[2])
        assert abs(area - want) <= 1e-9 * want

"""Generate the golden fixtures that pin the oracle (and, through it, the
GPU path) to the reference package itself.

Run HERE (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every case it stores the exact input arrays (so the fixtures do not
depend on the GPU box's numpy/libm, SURVEY.md finding 9) and what the
reference's public entry point returned:
  * vertices in discovery order (quickhull.py:186-188, :303-314),
  * iterations, discarded, warnings, or the exception class name,
  * the per-round trace (live points entering, kept, segments) recorded by
    wrapping seghull.quickhull.compact,
  * 3D: the loop candidates handed to _extreme_vertex_mask and its keep mask
    (quickhull.py:136-164).
Output: tests/golden/golden.npz (arrays) + tests/golden/golden.json (index).
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import seghull  # noqa: E402
import seghull.quickhull as QH  # noqa: E402
from seghull import Distribution, PointSet, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

_trace = []
_cands = []
_orig_compact = QH.compact
_orig_mask = QH._extreme_vertex_mask


def _compact(b, s):
    _trace.append((int(b.size), int(np.count_nonzero(b)), int(np.count_nonzero(s))))
    return _orig_compact(b, s)


def _mask(c, eps):
    keep = _orig_mask(c, eps)
    _cands.append((c.copy(), keep.copy()))
    return keep


QH.compact = _compact
QH._extreme_vertex_mask = _mask


def uniform_box(n, dim, seed):
    # "unit square" / "unit cube": raw splitmix64 uniforms (SURVEY.md finding 9)
    u = seghull.datagen._uniform_stream(seed, dim * n).reshape(n, dim)
    return PointSet(tuple(u[:, j].copy() for j in range(dim)))


def cases():
    out = []
    # reference KATs (test_quickhull.py)
    out.append(("kat-square-centre", PointSet.from_rows([(0, 0), (1, 0), (1, 1), (0, 1), (0.5, 0.5)])))
    out.append(("kat-single-2d", PointSet.from_rows([(2, 3)])))
    out.append(("kat-coincident-2d", PointSet.from_rows([(1, 1)] * 5)))
    out.append(("kat-collinear-2d", PointSet.from_rows([(i, 2 * i) for i in range(5)])))
    out.append(("kat-two-2d", PointSet.from_rows([(0, 0), (1, 5)])))
    out.append(("kat-duplicates-2d", PointSet.from_rows(
        [(0, 0), (1, 0), (1, 1), (0, 1), (1, 1), (0, 0), (0.5, 0.99)])))
    out.append(("kat-on-edge-2d", PointSet.from_rows(
        [(0, 0), (2, 0), (2, 2), (0, 2), (1, 0), (2, 1), (0, 1)])))
    cube = [(a, b, c) for a in (0, 1) for b in (0, 1) for c in (0, 1)]
    out.append(("kat-cube-centroid", PointSet.from_rows(cube + [(0.5, 0.5, 0.5)])))
    out.append(("kat-single-3d", PointSet.from_rows([(1, 2, 3)])))
    out.append(("kat-coincident-3d", PointSet.from_rows([(5, 5, 5)] * 4)))
    out.append(("kat-collinear-3d", PointSet.from_rows([(i, i, i) for i in range(6)])))
    out.append(("kat-coplanar-3d", PointSet.from_rows(
        [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (0.3, 0.4, 0)])))
    out.append(("kat-tetra", PointSet.from_rows([(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)])))
    out.append(("kat-triangle-3d", PointSet.from_rows([(0, 0, 0), (1, 0, 0), (0, 1, 0)])))
    out.append(("kat-two-3d", PointSet.from_rows([(0, 0, 0), (1, 2, 3)])))
    # distribution pins (test_quickhull.py:27-31, :98-102; acceptance crit 5)
    out.append(("on-circle-1024-s7", generate(Distribution("on-circle", 1024, 7))))
    out.append(("on-sphere-512-s3", generate(Distribution("on-sphere", 512, 3))))
    for kind in ("uniform-disk", "on-circle", "near-circle", "unit-square"):
        for n in (3, 5, 16, 100, 1000, 4000):
            for seed in (0, 1):
                pts = uniform_box(n, 2, seed) if kind == "unit-square" else \
                    generate(Distribution(kind, n, seed))
                out.append((f"{kind}-{n}-s{seed}", pts))
    for kind in ("uniform-ball", "on-sphere", "near-sphere", "unit-cube"):
        for n in (4, 8, 32, 100, 600, 2000):
            for seed in (0, 1):
                pts = uniform_box(n, 3, seed) if kind == "unit-cube" else \
                    generate(Distribution(kind, n, seed))
                out.append((f"{kind}-{n}-s{seed}", pts))
    out.extend(degenerate_3d())
    return out


def degenerate_3d():
    """Coplanar / cospherical 3D candidates, where the filter's eps rules
    decide (quickhull.py:136-164): lattices, points on the faces of a cube,
    Fibonacci spheres (every point on the sphere), two parallel rings."""
    out = []
    for k in (3, 4, 5, 7):
        g = np.arange(k, dtype=np.float64)
        z, y, x = np.meshgrid(g, g, g, indexing="ij")
        out.append((f"lattice-cube-{k}", PointSet((x.ravel().copy(), y.ravel().copy(), z.ravel().copy()))))
    rng = np.random.default_rng(11)
    for n in (300, 1500):
        u = rng.random((n, 2))
        face = rng.integers(0, 6, n)
        pts = np.empty((n, 3))
        for f in range(6):
            m = face == f
            ax, sgn = f // 2, float(f % 2)
            others = [a for a in range(3) if a != ax]
            pts[m, ax] = sgn
            pts[m, others[0]] = u[m, 0]
            pts[m, others[1]] = u[m, 1]
        out.append((f"cube-faces-{n}", PointSet(tuple(pts[:, j].copy() for j in range(3)))))
    for n in (200, 1000):
        i = np.arange(n, dtype=np.float64) + 0.5
        phi = np.arccos(1.0 - 2.0 * i / n)
        th = np.pi * (1.0 + 5.0 ** 0.5) * i
        out.append((f"fibonacci-sphere-{n}", PointSet((np.cos(th) * np.sin(phi), np.sin(th) * np.sin(phi),
                                                       np.cos(phi)))))
    t = np.linspace(0.0, 2.0 * np.pi, 60, endpoint=False)
    ring = np.concatenate([t, t])
    zz = np.concatenate([np.zeros(60), np.ones(60)])
    inner = rng.random((80, 3)) * 0.5 + 0.25
    out.append(("rings-120", PointSet((np.concatenate([np.cos(ring), inner[:, 0]]),
                                        np.concatenate([np.sin(ring), inner[:, 1]]),
                                        np.concatenate([zz, inner[:, 2]])))))
    return out


def main():
    arrays = {}
    index = []
    for i, (name, pts) in enumerate(cases()):
        _trace.clear()
        _cands.clear()
        fn = QH.quickhull_2d if pts.dim == 2 else QH.quickhull_3d
        rec = {"name": name, "key": f"c{i}", "dim": pts.dim, "n": pts.n}
        for j, c in enumerate(pts.coords):
            arrays[f"c{i}_in{j}"] = c
        try:
            r = fn(pts)
        except Exception as e:  # the exception class is part of the contract
            rec["error"] = type(e).__name__
        else:
            rec.update(iterations=r.iterations, discarded=r.discarded, warnings=list(r.warnings),
                       h=r.vertices.n)
            arrays[f"c{i}_verts"] = r.vertices.as_rows().reshape(-1, pts.dim)
        rec["trace"] = [list(t) for t in _trace]
        if _cands:
            c, keep = _cands[-1]
            arrays[f"c{i}_cand"] = c
            arrays[f"c{i}_keep"] = keep
        index.append(rec)
        print(name, rec.get("h"), rec.get("error", ""), len(_trace), flush=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "seghull 0.1.0 (/root/reference/pkg/src)",
                   "numpy": np.__version__, "cases": index}, f, indent=1)


if __name__ == "__main__":
    main()

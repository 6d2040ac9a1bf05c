"""Checks of a 3D facet list (test infrastructure, CPU).

A facet list of a convex hull is valid when
  * it is a closed, consistently oriented triangle mesh: every directed edge
    (i, j) occurs exactly once and its reverse (j, i) exactly once;
  * Euler: F = 2 V - 4 for the V vertices it references (a triangulated
    sphere);
  * every facet is a supporting plane, oriented outwards: for every input
    point s, det[[p_i 1] [p_j 1] [p_k 1] [s 1]] >= 0 (checked exactly in
    rational arithmetic for small inputs, with an fp64 error allowance for
    large ones);
and, on general-position inputs, the triangle set equals Qhull's simplices
(scipy.spatial.ConvexHull)."""

from collections import Counter
from fractions import Fraction

import numpy as np


def canonical(facets):
    """Set of vertex triples, order within a triple ignored."""
    return set(map(tuple, np.sort(np.asarray(facets, dtype=np.int64), axis=1).tolist()))


def check_mesh(facets):
    f = np.asarray(facets, dtype=np.int64)
    assert f.ndim == 2 and f.shape[1] == 3
    assert np.all(f[:, 0] != f[:, 1]) and np.all(f[:, 1] != f[:, 2]) and np.all(f[:, 0] != f[:, 2])
    edges = Counter()
    for a, b, c in f.tolist():
        edges[(a, b)] += 1
        edges[(b, c)] += 1
        edges[(c, a)] += 1
    assert max(edges.values()) == 1, "a directed edge is used twice"
    for (a, b) in edges:
        assert (b, a) in edges, f"edge ({a},{b}) has no twin"
    v = np.unique(f)
    assert len(f) == 2 * len(v) - 4, (len(f), len(v))
    assert len(canonical(f)) == len(f), "duplicate facet"
    return v


def check_supporting(rows, facets, exact=None, sample=2000):
    """Every point is on the inner side (or on the plane) of every facet
    (of a random sample of `sample` facets for large fp64 checks)."""
    rows = np.asarray(rows, dtype=np.float64)
    f = np.asarray(facets, dtype=np.int64)
    if exact is None:
        exact = len(rows) * len(f) <= 60_000
    if exact:
        R = [[Fraction(float(v)) for v in r] for r in rows]
        for a, b, c in f.tolist():
            A, B, C = R[a], R[b], R[c]
            u = [B[k] - A[k] for k in range(3)]
            w = [C[k] - A[k] for k in range(3)]
            n = [u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]]
            for s in R:
                # det4(a, b, c, s) = -n . (s - a) >= 0
                assert n[0] * (s[0] - A[0]) + n[1] * (s[1] - A[1]) + n[2] * (s[2] - A[2]) <= 0
        return
    if len(f) > sample:
        f = f[np.random.default_rng(0).choice(len(f), sample, replace=False)]
    a, b, c = rows[f[:, 0]], rows[f[:, 1]], rows[f[:, 2]]
    n = np.cross(b - a, c - a)
    scale = np.abs(n).sum(axis=1) * np.abs(rows).max() * 8
    for lo in range(0, len(f), 256):
        hi = min(len(f), lo + 256)
        d = np.einsum("fk,pk->fp", n[lo:hi], rows) - np.einsum("fk,fk->f", n[lo:hi], a[lo:hi])[:, None]
        assert np.all(d <= 1e-13 * scale[lo:hi, None]), "a point lies outside a facet"


def qhull_simplices(rows):
    from scipy.spatial import ConvexHull
    return ConvexHull(np.asarray(rows, dtype=np.float64)).simplices

"""Host self test of the exact orientation predicates behind the 3D facet
output (csrc/sh_exact.cuh, no GPU needed): the fp64 filter + expansion
arithmetic must give the sign of the exact determinant, and the Simulation
of Simplicity tie-break must equal the sign of the determinant of the
actually perturbed points, p[i][c] + eps^(2^(d*rank(i) + d-1-c)), evaluated
in rational arithmetic (eps small enough for the leading term to dominate)."""

import ctypes
import itertools
from fractions import Fraction

import numpy as np
import pytest

from paper_1201_2936_b200 import _lib


def orient(dim, pts, ids, exact_only=False):
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    nq = ids.shape[0]
    out = np.zeros(nq, np.int32)
    rc = _lib.lib().sh_orient_host(dim, pts.ctypes.data, ids.ctypes.data, nq, int(exact_only),
                                   out.ctypes.data)
    assert rc == 0
    return out


def det(m):
    m = [list(r) for r in m]
    n = len(m)
    d = Fraction(1)
    for c in range(n):
        p = next((r for r in range(c, n) if m[r][c] != 0), None)
        if p is None:
            return Fraction(0)
        if p != c:
            m[c], m[p] = m[p], m[c]
            d = -d
        d *= m[c][c]
        for r in range(c + 1, n):
            f = m[r][c] / m[c][c]
            for k in range(c, n):
                m[r][k] -= f * m[c][k]
    return d


def exact_sign(dim, pts):
    m = [[Fraction(float(v)) for v in p] + [Fraction(1)] for p in pts]
    return int(np.sign(det(m)))


def sos_sign(dim, pts, ids, eps=Fraction(1, 2 ** 16)):
    rank = {g: r for r, g in enumerate(sorted(ids))}
    m = []
    for p, g in zip(pts, ids):
        r = rank[g]
        m.append([Fraction(float(v)) + eps ** (2 ** (dim * r + dim - 1 - c)) for c, v in enumerate(p)]
                 + [Fraction(1)])
    return int(np.sign(det(m)))


@pytest.mark.parametrize("dim", [2, 3])
def test_random_inputs_match_exact_sign(dim):
    rng = np.random.default_rng(5)
    nq = 400
    pts = rng.random((nq, dim + 1, dim))
    # near-degenerate: last point almost on the hyperplane of the others
    w = rng.random((nq, dim))
    w /= w.sum(axis=1, keepdims=True)
    near = np.einsum("qk,qkc->qc", w, pts[:, :dim, :]) + rng.normal(0, 1e-15, (nq, dim))
    pts[nq // 2:, dim] = near[nq // 2:]
    ids = np.tile(np.arange(dim + 1), (nq, 1))
    got = orient(dim, pts.reshape(nq, -1), ids)
    want = []
    for q in range(nq):
        s = exact_sign(dim, pts[q])
        want.append(s if s else sos_sign(dim, pts[q], ids[q]))
    assert np.array_equal(got, np.array(want))


@pytest.mark.parametrize("dim", [2, 3])
def test_degenerate_inputs_match_perturbed_determinant(dim):
    rng = np.random.default_rng(11)
    nq = 300
    # small integer lattice: many exactly collinear / coplanar / coincident rows
    pts = rng.integers(-2, 3, size=(nq, dim + 1, dim)).astype(np.float64)
    ids = np.array([rng.permutation(50)[:dim + 1] for _ in range(nq)], dtype=np.int64)
    got = orient(dim, pts.reshape(nq, -1), ids)
    got_exact = orient(dim, pts.reshape(nq, -1), ids, exact_only=True)
    want = np.array([sos_sign(dim, pts[q], ids[q]) for q in range(nq)])
    assert np.array_equal(got, want)
    assert np.array_equal(got_exact, want)
    assert np.all(got != 0)


def test_sos_is_antisymmetric_and_consistent():
    rng = np.random.default_rng(3)
    for _ in range(100):
        pts = rng.integers(0, 2, size=(4, 3)).astype(np.float64)
        ids = rng.permutation(20)[:4].astype(np.int64)
        base = orient(3, pts.reshape(1, -1), ids.reshape(1, -1))[0]
        for perm in itertools.permutations(range(4)):
            perm = list(perm)
            inv = sum(1 for i in range(4) for j in range(i + 1, 4) if perm[i] > perm[j])
            s = orient(3, pts[perm].reshape(1, -1), ids[perm].reshape(1, -1))[0]
            assert s == base * (-1) ** inv

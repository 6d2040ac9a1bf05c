"""CPU: the facet checker itself (tests/facet_check.py) accepts Qhull's
triangulations and rejects broken ones."""

import numpy as np
import pytest

from facet_check import canonical, check_mesh, check_supporting, qhull_simplices


def oriented_qhull(rows):
    s = qhull_simplices(rows)
    c = rows.mean(axis=0)
    a, b, d = rows[s[:, 0]], rows[s[:, 1]], rows[s[:, 2]]
    n = np.cross(b - a, d - a)
    flip = np.einsum("fk,fk->f", n, c - a) > 0
    s[flip] = s[flip][:, [0, 2, 1]]
    return s


def test_checker_accepts_qhull_and_rejects_broken():
    rng = np.random.default_rng(0)
    rows = rng.normal(size=(300, 3))
    f = oriented_qhull(rows)
    check_mesh(f)
    check_supporting(rows, f, exact=True)
    check_supporting(rows, f, exact=False)
    with pytest.raises(AssertionError):
        check_mesh(f[1:])
    g = f.copy()
    g[0] = g[0][[0, 2, 1]]
    with pytest.raises(AssertionError):
        check_mesh(g)
    with pytest.raises(AssertionError):
        check_supporting(rows, f[:, [0, 2, 1]], exact=True)
    assert canonical(f) == canonical(qhull_simplices(rows))

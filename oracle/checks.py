"""ORACLE -- test infrastructure only (see oracle/__init__.py).

Sequential restatement of the reference's brute-force checks used by the
CLI's `verify` (/root/reference/pkg/src/seghull/oracle.py):
  giftwrap2d   hull2_giftwrap, oracle.py:20-52 (plain sequential scan)
  bruteforce3d hull3_bruteforce, oracle.py:82-118 (vertex set)
Pinned to the reference's own outputs by tests/test_checks.py
(tests/golden/golden_checks.json, made by tests/golden/make_golden_checks.py)."""

import itertools

import numpy as np


def giftwrap2d(x, y, eps):
    """Indices (first occurrence of each coordinate pair) of the strict hull,
    CCW from the lexicographic minimum; the scan order and replacement rule
    of hull2_giftwrap."""
    pts = list(zip(map(float, x), map(float, y)))
    first = {}
    for i, p in enumerate(pts):
        first.setdefault(p, i)
    start = min(pts)
    hull = [start]
    cur = start
    for _ in range(len(pts) + 1):
        cx, cy = cur
        cand = None
        for q in pts:
            if q == cur:
                continue
            if cand is None:
                cand = q
                continue
            cross = (cand[0] - cx) * (q[1] - cy) - (cand[1] - cy) * (q[0] - cx)
            limit = eps * float(np.hypot(cand[0] - cx, cand[1] - cy))
            if cross < -limit:
                cand = q
            elif cross <= limit:
                if (q[0] - cx) ** 2 + (q[1] - cy) ** 2 > (cand[0] - cx) ** 2 + (cand[1] - cy) ** 2:
                    cand = q
        if cand is None or cand == start:
            break
        hull.append(cand)
        cur = cand
    return [first[p] for p in hull]


def bruteforce3d(rows, eps):
    """Sorted indices of the points that are corners of a supporting,
    non-straight triple (hull3_bruteforce's vertex set, before dedup by
    coordinates)."""
    rows = np.asarray(rows, np.float64)
    n = rows.shape[0]
    out = set()
    for i, j, k in itertools.combinations(range(n), 3):
        a, b, c = rows[i], rows[j], rows[k]
        nrm = np.cross(b - a, c - a)
        nl = np.linalg.norm(nrm)
        if nl <= eps * (np.linalg.norm(b - a) + np.linalg.norm(c - a)):
            continue
        d = rows @ nrm - nrm @ a
        if (d >= -eps * nl).all() or (d <= eps * nl).all():
            out.update((i, j, k))
    return sorted(out)

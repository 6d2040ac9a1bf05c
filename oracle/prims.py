"""ORACLE -- test infrastructure only (see oracle/__init__.py).

Sequential restatement of the reference's framework primitives
(/root/reference/pkg/src/seghull/segments.py:201-266,
primitives.py:91-148): plain loops, no scans.  Pinned to the reference's
own outputs by tests/test_primitives.py (tests/golden/golden_prims.npz)."""

import numpy as np

_IDENT_I = {"sum": 0, "max": np.iinfo(np.int64).min, "min": np.iinfo(np.int64).max}
_IDENT_F = {"max": -np.inf, "min": np.inf}


def segmented_scan(values, heads, op, direction="forward", mode="inclusive"):
    v = np.asarray(values)
    floating = np.issubdtype(v.dtype, np.floating)
    v = v.astype(np.float64) + 0.0 if floating else v.astype(np.int64)
    h = np.asarray(heads, dtype=bool)
    n = v.size
    order = range(n) if direction == "forward" else range(n - 1, -1, -1)
    ident = (_IDENT_F if floating else _IDENT_I)[op]
    out = np.empty_like(v)
    acc = ident
    prev = None
    for i in order:
        # start of a segment in the scan direction
        start = (prev is None) or (h[i] if direction == "forward" else h[prev])
        if start:
            acc = ident
        before = acc
        if op == "sum":
            acc = acc + v[i]
        elif op == "max":
            acc = max(acc, v[i])
        else:
            acc = min(acc, v[i])
        out[i] = before if mode == "exclusive" else acc
        prev = i
    return out


def flag_permute(f, heads, k):
    """Per-segment stable counting sort by state; new heads per group."""
    f = np.asarray(f, dtype=np.int64)
    h = np.asarray(heads, dtype=bool)
    n = f.size
    p = np.empty(n, np.int64)
    s_new = np.zeros(n, bool)
    starts = list(np.flatnonzero(h)) + [n]
    for a, b in zip(starts[:-1], starts[1:]):
        pos = a
        for j in range(k):
            members = [i for i in range(a, b) if f[i] == j]
            if members:
                s_new[pos] = True
            for i in members:
                p[i] = pos
                pos += 1
    return p, s_new


def compact(b, heads):
    b = np.asarray(b, dtype=bool)
    h = np.asarray(heads, dtype=bool)
    n = b.size
    p = np.empty(n, np.int64)
    c = 0
    for i in range(n):
        p[i] = c
        c += int(b[i])
    s_new = np.zeros(c, bool)
    starts = list(np.flatnonzero(h)) + [n]
    for a, e in zip(starts[:-1], starts[1:]):
        kept = [i for i in range(a, e) if b[i]]
        if kept:
            s_new[p[kept[0]]] = True
    return p, c, s_new

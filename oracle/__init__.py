"""ORACLE -- test infrastructure only (never imported by the product package).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / CPU baseline.

ctypes front-end for ``qh_oracle.c``, the plain-C restatement of the
reference drivers ``quickhull_2d`` / ``quickhull_3d``
(/root/reference/pkg/src/seghull/quickhull.py:167-279, :282-446).  The 3D
post-loop filter of the reference (``_extreme_vertex_mask``,
quickhull.py:136-164: dgemm certificate + eps supporting planes + HiGHS LP)
is not bit-reproducible off the reference's BLAS/LP; ``extreme_filter_qhull``
substitutes the exact extreme-point set via Qhull (scipy), which SURVEY.md
Appendix A.6 found equal to the reference's output on every tested 3D input.
Its parity with the reference on the golden inputs is checked in
tests/test_oracle.py.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libqh_oracle.so")
_lib = None

STATUS_OK = 0
STATUS_EMPTY = 2
STATUS_DEGENERATE = 3
STATUS_ROUND_GUARD = 4
WARN_COLLINEAR = 1

_p = ctypes.c_void_p
_i64 = ctypes.c_int64


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "qh_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oq_hull2d.restype = ctypes.c_int
        L.oq_hull2d.argtypes = [_p, _p, _i64, ctypes.c_double, ctypes.c_double, _p, _p, _p, _p, _p,
                                _i64, _p]
        L.oq_hull3d.restype = ctypes.c_int
        L.oq_hull3d.argtypes = [_p, _p, _p, _i64, ctypes.c_double, ctypes.c_double, _p, _p, _p, _p,
                                _p, _p, _i64, _p, _i64, _p]
        L.oq_giftwrap2d.restype = _i64
        L.oq_giftwrap2d.argtypes = [_p, _p, _i64, ctypes.c_double, _p, _i64]
        _lib = L
    return _lib


def giftwrap2d(x, y, eps):
    """hull2_giftwrap (reference seghull/oracle module lines 20-52) in C:
    indices (first occurrence per coordinate pair), CCW from the
    lexicographic minimum.  Pinned to the reference by tests/test_checks.py."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty(x.size + 1, dtype=np.int64)
    h = lib().oq_giftwrap2d(_ptr(x), _ptr(y), x.size, float(eps), _ptr(out), out.size)
    if h < 0:
        raise ValueError("giftwrap2d: bad arguments")
    return out[:h]


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleResult:
    """Loop output of the restated reference driver.

    idx       original indices of the vertices (3D: loop candidates) in the
              reference's discovery order
    iterations, flags, status, trace (rounds x [live, kept, nseg]),
    flat_counts (3D, per round), filter (3D: 1 when the reference would run
    its candidate filter)
    """

    def __init__(self, **kw):
        self.__dict__.update(kw)


def hull2d(x, y, eps_rel=1e-12, trace_cap=4096, eps_abs=float("nan")):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = x.size
    out = np.zeros(max(n, 1), np.int64)
    h, it, tl = (np.zeros(1, np.int64) for _ in range(3))
    fl = np.zeros(1, np.int32)
    tr = np.zeros((trace_cap, 3), np.int64)
    st = lib().oq_hull2d(_ptr(x), _ptr(y), n, eps_rel, eps_abs, _ptr(out), _ptr(h), _ptr(it), _ptr(fl),
                         _ptr(tr), trace_cap, _ptr(tl))
    return OracleResult(status=st, idx=out[:h[0]].copy(), iterations=int(it[0]),
                        flags=int(fl[0]), trace=tr[:tl[0]].copy(), filter=0,
                        flat_counts=np.zeros(0, np.int64))


def hull3d(x, y, z, eps_rel=1e-12, trace_cap=4096, eps_abs=float("nan")):
    x, y, z = (np.ascontiguousarray(c, dtype=np.float64) for c in (x, y, z))
    n = x.size
    out = np.zeros(max(n, 1), np.int64)
    h, it, tl = (np.zeros(1, np.int64) for _ in range(3))
    fl = np.zeros(1, np.int32)
    filt = np.zeros(1, np.int32)
    flat = np.zeros(trace_cap, np.int64)
    tr = np.zeros((trace_cap, 3), np.int64)
    st = lib().oq_hull3d(_ptr(x), _ptr(y), _ptr(z), n, eps_rel, eps_abs, _ptr(out), _ptr(h), _ptr(it),
                         _ptr(fl), _ptr(filt), _ptr(flat), trace_cap, _ptr(tr), trace_cap, _ptr(tl))
    iters = int(it[0])
    return OracleResult(status=st, idx=out[:h[0]].copy(), iterations=iters, flags=int(fl[0]),
                        trace=tr[:tl[0]].copy(), filter=int(filt[0]),
                        flat_counts=flat[:min(iters, trace_cap)].copy())


def extreme_filter_qhull(rows):
    """Mask of candidate rows that are vertices of their convex hull (Qhull).

    Substitute for the reference's _extreme_vertex_mask (quickhull.py:136-164)
    with the same m <= 4 shortcut (:148-149)."""
    m = rows.shape[0]
    if m <= 4:
        return np.ones(m, dtype=bool)
    from scipy.spatial import ConvexHull
    hull = ConvexHull(rows)
    mask = np.zeros(m, dtype=bool)
    mask[hull.vertices] = True
    return mask


def warnings_2d(res, n):
    if res.flags & WARN_COLLINEAR:
        return ["collinear input: hull is the two x-extrema"]
    return []


def warnings_3d(res, pruned):
    """Reference warning strings (quickhull.py:308-310, :338, :387-389)."""
    w = []
    if res.flags & WARN_COLLINEAR:
        w.append("collinear input: hull is the two extrema")
    for r, m in enumerate(res.flat_counts, start=1):
        if m:
            w.append(f"round {r}: dropped {int(m)} near-coplanar segment(s)")
    if pruned:
        w.append(f"pruned {pruned} non-extreme candidate vertex(es) emitted by incomplete "
                 "per-face outside sets")
    return w


def full_hull3d(x, y, z, eps_rel=1e-12, eps_abs=float("nan")):
    """Loop candidates + Qhull filter: the reference-equivalent 3D result
    (indices in the reference's order) for inputs where the reference's own
    LP filter is infeasible."""
    r = hull3d(x, y, z, eps_rel, eps_abs=eps_abs)
    if r.status != STATUS_OK:
        return r, r.idx, []
    idx = r.idx
    pruned = 0
    if r.filter and idx.size:
        rows = np.column_stack([np.asarray(x)[idx], np.asarray(y)[idx], np.asarray(z)[idx]])
        keep = extreme_filter_qhull(rows)
        pruned = int((~keep).sum())
        idx = idx[keep]
    return r, idx, warnings_3d(r, pruned)

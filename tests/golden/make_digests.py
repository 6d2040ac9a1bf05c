"""Full-size reference digests for the BASELINE configs the reference can
run here (C1, C2, C3, C3', C4-cube; minutes each).

Run HERE (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_digests.py

For each config it runs the reference's public entry point on the full
cloud (same generators and seeds as bench.py) and stores, in
tests/golden/digests.json:
  * n, hull size, iterations, discarded, warnings,
  * sha256 of the sorted original indices of the vertices (int64 LE) --
    indices recovered from the returned coordinates (every input point is
    distinct in these clouds),
  * sha256 of vertices.as_rows().tobytes() in the reference's discovery
    order (quickhull.py:186-188),
  * the per-round trace (live points entering, kept, segments) recorded by
    wrapping seghull.quickhull.compact.
The GPU tests (tests/test_gpu_digests.py) compare the device hull with
these on the GPU box, where the reference is not available.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import seghull  # noqa: E402
import seghull.quickhull as QH  # noqa: E402
from seghull import Distribution, PointSet, generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
_trace = []
_orig_compact = QH.compact


def _compact(b, s):
    _trace.append((int(b.size), int(np.count_nonzero(b)), int(np.count_nonzero(s))))
    return _orig_compact(b, s)


QH.compact = _compact


def uniform_box(n, dim, seed):
    u = seghull.datagen._uniform_stream(seed, dim * n).reshape(n, dim)
    return PointSet(tuple(u[:, j].copy() for j in range(dim)))


CONFIGS = {
    "C1": lambda: uniform_box(1_000_000, 2, 0),
    "C2": lambda: generate(Distribution("uniform-disk", 100_000_000, 0)),
    "C3": lambda: generate(Distribution("on-circle", 10_000_000, 0)),
    "C3n": lambda: generate(Distribution("near-circle", 10_000_000, 0, band=0.01)),
    "C4c": lambda: uniform_box(10_000_000, 3, 0),
}


def indices_of(points, verts):
    """Original indices of the vertex rows (distinct input points)."""
    cols = points.coords
    order = np.lexsort(tuple(reversed(cols)))
    keys = np.rec.fromarrays([c[order] for c in cols])
    vk = np.rec.fromarrays(list(verts.coords))
    pos = np.searchsorted(keys, vk)
    idx = order[pos]
    for c, v in zip(cols, verts.coords):
        assert np.array_equal(c[idx], v), "vertex not found in the input"
    return idx


def main(names):
    seghull.parallel.set_workers(os.cpu_count())
    path = os.path.join(HERE, "digests.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        pts = CONFIGS[name]()
        _trace.clear()
        t0 = time.time()
        f = QH.quickhull_2d if pts.dim == 2 else QH.quickhull_3d
        r = f(pts)
        dt = time.time() - t0
        idx = indices_of(pts, r.vertices)
        out[name] = {
            "n": int(pts.n), "dim": int(pts.dim), "h": int(r.vertices.n), "iterations": int(r.iterations),
            "discarded": int(r.discarded), "warnings": list(r.warnings),
            "sorted_idx_sha256": hashlib.sha256(np.sort(idx).astype("<i8").tobytes()).hexdigest(),
            "rows_sha256": hashlib.sha256(r.vertices.as_rows().tobytes()).hexdigest(),
            "trace": [list(t) for t in _trace],
            "reference_seconds": round(dt, 1),
        }
        print(name, out[name]["h"], out[name]["iterations"], round(dt, 1), "s", flush=True)
        json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))

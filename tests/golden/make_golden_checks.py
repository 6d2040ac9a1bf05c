"""Golden vectors for the `verify` brute-force checks, from the reference's
own oracles (seghull.oracle.hull2_giftwrap / hull3_bruteforce).

Run HERE (the reference is importable only in the build container):

    python tests/golden/make_golden_checks.py

Writes tests/golden/golden_checks.json: per case the input rows, eps
(Tolerance().effective) and the reference's output coordinates."""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from seghull import Distribution, PointSet, Tolerance, generate  # noqa: E402
from seghull.oracle import hull2_giftwrap, hull3_bruteforce  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cases():
    for kind, n, seed in (("uniform-disk", 300, 1), ("on-circle", 64, 2), ("near-circle", 200, 4),
                          ("uniform-disk", 1, 0), ("uniform-disk", 2, 3)):
        yield kind, generate(Distribution(kind, n, seed=seed))
    g = np.arange(6, dtype=np.float64)
    X, Y = np.meshgrid(g, g)  # collinear boundary points, interior of edges dropped
    yield "grid6", PointSet((X.ravel().copy(), Y.ravel().copy()))
    r = np.random.default_rng(7).random((40, 2))
    r = np.concatenate([r, r[:10]])  # duplicates
    yield "dups", PointSet((r[:, 0].copy(), r[:, 1].copy()))
    c = np.random.default_rng(8).random((50, 3))
    yield "cube-corners", PointSet(tuple(np.concatenate([c, np.array(np.meshgrid([0., 1], [0., 1], [0., 1])).reshape(3, -1).T])[:, k].copy() for k in range(3)))
    for kind, n, seed in (("uniform-ball", 48, 9), ("on-sphere", 30, 1), ("near-sphere", 60, 2)):
        yield kind, generate(Distribution(kind, n, seed=seed))


def main():
    out = []
    for name, ps in cases():
        tol = Tolerance()
        eps = tol.effective(ps)
        res = hull2_giftwrap(ps, tol) if ps.dim == 2 else hull3_bruteforce(ps, tol)
        out.append({"name": name, "dim": ps.dim, "eps": eps, "rows": ps.as_rows().tolist(),
                    "hull": res.as_rows().tolist()})
    with open(os.path.join(HERE, "golden_checks.json"), "w") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out)} cases")


if __name__ == "__main__" and "--big" not in sys.argv:
    main()


def big():
    """Digest of the sequential gift wrap on a dense circle (100k points, all
    on the boundary, many within-eps ties), from the C restatement
    (oracle.giftwrap2d, pinned to hull2_giftwrap by tests/test_checks.py);
    the Python reference would need hours here.  ~2 min.

        python tests/golden/make_golden_checks.py --big"""
    import hashlib
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    import oracle
    out = []
    for kind, n, seed in (("on-circle", 100000, 1),):
        ps = generate(Distribution(kind, n, seed=seed))
        eps = Tolerance().effective(ps)
        idx = oracle.giftwrap2d(ps.coords[0], ps.coords[1], eps).astype("<i8")
        out.append({"kind": kind, "n": n, "seed": seed, "eps": eps, "h": int(idx.size),
                    "sha256": hashlib.sha256(idx.tobytes()).hexdigest()})
    with open(os.path.join(HERE, "golden_checks_big.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__" and "--big" in sys.argv:
    big()

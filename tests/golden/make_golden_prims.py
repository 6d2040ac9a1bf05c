"""Golden vectors for the framework primitives, produced by the reference
itself (segments.py / primitives.py).  Run HERE:

    python tests/golden/make_golden_prims.py

Stores inputs and outputs of segmented_scan (all 12 specs, int64 and
float64 with -0.0 / ties), flag_permute (k = 1, 2, 3), compact and the
paper's Figure 1 example into tests/golden/golden_prims.npz.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from seghull import ScanSpec, compact, flag_permute, segmented_scan  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def heads(rng, n, density):
    s = rng.random(n) < density
    if n:
        s[0] = True
    return s


def main():
    rng = np.random.default_rng(2024)
    out = {}
    cases = []
    for ci, (n, dens) in enumerate([(1, 0.5), (7, 0.3), (100, 0.15), (5000, 0.15), (3000, 0.001),
                                    (20_000, 0.02)]):
        s = heads(rng, n, dens)
        vi = rng.integers(-50, 50, n)
        vf = np.round(rng.standard_normal(n), 2)
        if n > 3:
            vf[::7] = -0.0
        out[f"s{ci}_heads"] = s
        out[f"s{ci}_vi"] = vi
        out[f"s{ci}_vf"] = vf
        for op in ("sum", "max", "min"):
            for d in ("forward", "backward"):
                for m in ("inclusive", "exclusive"):
                    spec = ScanSpec(op, d, m)
                    out[f"s{ci}_{op}_{d}_{m}_i"] = segmented_scan(vi, s, spec)
                    if op != "sum":
                        out[f"s{ci}_{op}_{d}_{m}_f"] = segmented_scan(vf, s, spec)
        for k in (1, 2, 3):
            f = rng.integers(0, k, n)
            pm, s2 = flag_permute(f, s, k)
            out[f"s{ci}_fp{k}_f"] = f
            out[f"s{ci}_fp{k}_p"] = pm.p
            out[f"s{ci}_fp{k}_s"] = s2
        b = rng.random(n) < 0.4
        pm, s2 = compact(b, s)
        out[f"s{ci}_cp_b"] = b
        out[f"s{ci}_cp_p"] = pm.p
        out[f"s{ci}_cp_len"] = np.array([pm.out_len])
        out[f"s{ci}_cp_s"] = s2
        cases.append(ci)
    out["ncases"] = np.array([len(cases)])
    np.savez_compressed(os.path.join(HERE, "golden_prims.npz"), **out)


if __name__ == "__main__":
    main()

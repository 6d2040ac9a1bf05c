"""Debug: forced long rounds on one input; print the per-round trace vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
kind, n, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cols = generate(kind, n, seed)
o = oracle.hull2d(*cols) if len(cols) == 2 else oracle.hull3d(*cols)
try:
    f = P.hull_indices_2d if len(cols) == 2 else P.hull_indices_3d
    idx, res = f(tuple(torch.from_numpy(c).cuda() for c in cols), return_info=True)
    tr = P.trace()
    print("ours", idx.numel(), res.iterations, "oracle", len(o.idx), o.iterations)
    for r in range(max(len(tr), len(o.trace))):
        a = tr[r].tolist() if r < len(tr) else None
        b = o.trace[r].tolist() if r < len(o.trace) else None
        print(r + 1, a, b, "" if a is not None and b is not None and a[:3] == b[:3] else "<<<")
except Exception as e:
    print("ERR", e)

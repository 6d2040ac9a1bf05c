"""C5 at full size on one GPU: single hull vs 8-way loopback sharding, and
the loop against the oracle (candidates, rounds)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import oracle
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import sharded
from paper_1201_2936_b200.datagen import generate
t = time.time()
cols = generate("uniform-ball", 200_000_000, 0)
print("gen s", time.time() - t, flush=True)
d = tuple(torch.from_numpy(c).cuda() for c in cols)
idx, _, res = P.hull_indices_3d(d, return_info=True)
torch.cuda.synchronize()
print("single: h", res.h, "cand", res.candidates, "rounds", res.iterations, flush=True)
for p in (8,):
    t = time.time()
    g, info = sharded.hull_sharded_loopback(d, p, return_info=True)
    torch.cuda.synchronize()
    print("loopback", p, "h", g.numel(), "union", info["union"], "equal", np.array_equal(np.sort(g.cpu().numpy()), np.sort(idx.cpu().numpy())), "s", time.time() - t, flush=True)
t = time.time()
o = oracle.hull3d(*cols)
print("oracle loop s", time.time() - t, "cand", len(o.idx), "rounds", o.iterations, flush=True)
print("loop equal", res.candidates == len(o.idx) and res.iterations == o.iterations, flush=True)
from scipy.spatial import ConvexHull
rows = np.column_stack([c[o.idx] for c in cols])
hv = o.idx[ConvexHull(rows).vertices]
print("qhull(candidates) equal", np.array_equal(np.sort(hv), np.sort(idx.cpu().numpy())), flush=True)

import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
n = 2_000_000
cols = generate("uniform-ball", n, 0)
d = tuple(torch.from_numpy(c).cuda() for c in cols)
full = P.hull_indices_3d(d)
print("full", full.numel(), {k: v for k, v in P.filter_stats().items() if not k.startswith("item")})
R = 4
for r in range(R):
    p = P.hull_indices_3d(d, filter_share=(r, R))
    fs = P.filter_stats()
    extra = p[~torch.isin(p, full)]
    print(r, p.numel(), {k: fs[k] for k in ("candidates", "ambiguous", "gjk_capped", "certified", "local_pruned", "local_extreme", "global_gjk")}, "extra-vs-full", extra.numel())
# repeat the full run twice more
for _ in range(2):
    f2 = P.hull_indices_3d(d)
    print("full again equal", torch.equal(f2, full))

import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import sharded
from paper_1201_2936_b200.datagen import generate
for n in (2_000_000, 20_000_000):
    cols = generate("uniform-ball", n, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    full = np.sort(P.hull_indices_3d(d).cpu().numpy())
    for ns in (2, 4, 8):
        for split in (False, True):
            g = sharded.hull_sharded_loopback(d, ns, split_merge=split)
            g = np.sort(g.cpu().numpy())
            print(n, ns, split, len(full), len(g), np.array_equal(g, full), len(np.setdiff1d(full, g)), len(np.setdiff1d(g, full)))
    # direct shares on the whole input
    for R in (2, 4, 8):
        parts = [P.hull_indices_3d(d, filter_share=(r, R)) for r in range(R)]
        keep = torch.ones(parts[0].numel(), dtype=torch.bool, device="cuda")
        for p in parts[1:]:
            keep &= torch.isin(parts[0], p)
        print("direct", n, R, len(full), int(keep.sum()), np.array_equal(np.sort(parts[0][keep].cpu().numpy()), full), [p.numel() for p in parts])

"""3D filter diagnostics + per-kernel times (launch mode 2)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from paper_1201_2936_b200.datagen import generate

L = _lib.lib()
names = ["init", "first_reduce", "line_far", "round_first", "round", "book", "filter", "output", "facets"]
for kind, n in [("unit-cube", 10_000_000), ("uniform-ball", 10_000_000), ("uniform-ball", 200_000_000)]:
    cols = generate(kind, n, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    del cols
    idx = P.hull_indices_3d(d)
    ctx = _lib.context(0)
    L.sh_set_launch_mode(ctx, 2)
    idx = P.hull_indices_3d(d)
    torch.cuda.synchronize()
    kinds = np.zeros(4096, np.int32); ms = np.zeros(4096, np.float32)
    k = L.sh_launch_times(ctx, kinds.ctypes.data, ms.ctypes.data, 4096)
    L.sh_set_launch_mode(ctx, 0)
    st = np.zeros(15, np.int64)
    L.sh_filter_stats(ctx, st.ctypes.data, 15)
    tr = P.trace()
    by = {names[i]: round(float(ms[:k][kinds[:k] == i].sum()), 3) for i in sorted(set(kinds[:k].tolist()))}
    rounds = [round(float(x), 3) for x in ms[:k][kinds[:k] == 4]]
    print(f"{kind} {n}: h={idx.numel()} {by}")
    print("  rounds ms:", rounds)
    print("  trace (live, kept, nseg):", tr[:, :3].tolist())
    print("  filter m=%d G=%d amb=%d capped=%d certified=%d queries=%d scanned=%d gjk_iters=%d local_in=%d local_out=%d fallback=%d" % tuple(st[:11]))
    cy = st[11:15].astype(float)
    print("  cycles: cert %.3g local %.3g out %.3g fallback %.3g  (per cand: cert %.0f)" % (*cy, cy[0] / max(st[0], 1)))
    del d
    torch.cuda.empty_cache()

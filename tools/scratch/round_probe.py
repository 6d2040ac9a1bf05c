"""Per-launch device times (launch mode 2) and per-round bytes for a config."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from paper_1201_2936_b200.datagen import generate

L = _lib.lib()
names = ["init", "first_reduce", "line_far", "round_first", "round", "book", "filter", "output", "facets"]
cfgs = [("uniform-disk", 100_000_000), ("on-circle", 10_000_000), ("uniform-ball", 10_000_000)]
if len(sys.argv) > 1:
    cfgs = [c for c in cfgs if c[0] in sys.argv[1:]]
for kind, n in cfgs:
    cols = generate(kind, n, 0)
    dim = len(cols)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    del cols
    f = P.hull_indices_2d if dim == 2 else P.hull_indices_3d
    f(d)
    ctx = _lib.context(0)
    L.sh_set_launch_mode(ctx, 2)
    best = None
    for _ in range(3):
        f(d)
        torch.cuda.synchronize()
        kinds = np.zeros(4096, np.int32); ms = np.zeros(4096, np.float32)
        k = L.sh_launch_times(ctx, kinds.ctypes.data, ms.ctypes.data, 4096)
        if best is None or ms[:k].sum() < best[1].sum():
            best = (kinds[:k].copy(), ms[:k].copy())
    L.sh_set_launch_mode(ctx, 0)
    kinds, ms = best
    tr = P.trace()
    Rd = 8 * dim + 4
    rt = ms[(kinds == 3) | (kinds == 4)]
    byts = [8 * dim * n] + [(8 * dim * n if r == 0 else Rd * int(a)) + Rd * int(b) for r, (a, b, _, _) in enumerate(tr)]
    print(f"{kind} {n}: total {ms.sum():.3f} ms", {names[i]: round(float(ms[kinds == i].sum()), 3) for i in sorted(set(kinds.tolist()))})
    for r, (t, b) in enumerate(zip(rt, byts)):
        live = int(tr[r - 1][0]) if r else n
        segs = int(tr[r - 1][2]) if r else 1
        print(f"  round {r}: {t*1e3:8.1f} us  live {live:>11,} segs {segs:>8,}  {b/1e9:7.3f} GB  {b/(t*1e-3)/1e9:7.1f} GB/s")
    books = ms[kinds == 5]
    print("  book us:", [round(float(x) * 1e3, 1) for x in books])
    del d
    torch.cuda.empty_cache()

"""Facet-build diagnostics on the GPU: time + counters per config."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from paper_1201_2936_b200.datagen import generate

for kind, n in [("unit-cube", 10_000_000), ("uniform-ball", 10_000_000), ("uniform-ball", 1_000_000),
                ("on-sphere", 200_000)]:
    cols = generate(kind, n, 0)
    d = tuple(torch.from_numpy(c).cuda() for c in cols)
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        i0 = P.hull_indices_3d(d)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        idx, fac = P.hull_indices_3d(d, facets=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
    st = np.zeros(9, np.int64)
    _lib.lib().sh_facet_stats(_lib.context(0), st.ctypes.data, 9)
    print(f"{kind} {n}: h={idx.numel()} F={fac.shape[0]} verts {1e3*(t1-t):.2f} ms, +facets {1e3*(t2-t1):.2f} ms;"
          f" items={st[1]} queries={st[2]} batches={st[3]} beat={st[4]} nodes={st[5]}"
          f" wrap_cyc/q={st[6]/max(st[2],1):.0f} wait_cyc={st[7]:.3g} init_cyc={st[8]}", flush=True)

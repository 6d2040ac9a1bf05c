"""Filter diagnostics: time + counters of the 3D extreme filter."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from paper_1201_2936_b200.datagen import generate
L, ctx = _lib.lib(), _lib.context(0)
for kind, n in [("uniform-ball", 10**6), ("uniform-ball", 10**7), ("unit-cube", 10**7), ("near-sphere", 10**6), ("uniform-ball", 10**8)]:
    d = tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 0))
    P.hull_indices_3d(d)
    L.sh_set_launch_mode(ctx, 2)
    idx, _, res = P.hull_indices_3d(d, return_info=True)
    L.sh_set_launch_mode(ctx, 0)
    kinds = np.zeros(256, np.int32); ms = np.zeros(256, np.float32)
    k = L.sh_launch_times(ctx, kinds.ctypes.data, ms.ctypes.data, 256)
    st = np.zeros(11, np.int64); L.sh_filter_stats(ctx, st.ctypes.data, 11)
    print(kind, n, "cand", res.candidates, "h", res.h, "filter ms", float(ms[:k][kinds[:k] == 6].sum()),
          "stats m,G,amb,capped,cert0,queries,scanned,iters,loc_in,loc_out,fallback =", st.tolist(), flush=True)

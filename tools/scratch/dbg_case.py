import sys, json
import numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from golden_io import load
name = sys.argv[1]
c = next(c for c in load() if c.name == name)
L, ctx = _lib.lib(), _lib.context(0)
L.sh_set_launch_mode(ctx, int(__import__("os").environ.get("SH_MODE", "0")))
d = tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in c.coords)
f = P.hull_indices_2d if c.dim == 2 else P.hull_indices_3d
print(name, f(d), flush=True)

"""Profiling driver: one warm-up hull + one measured hull on a resident input."""
import sys, argparse
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="uniform-disk")
ap.add_argument("--n", type=int, default=10**8)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--hostloop", type=int, default=1)
a = ap.parse_args()
import paper_1201_2936_b200._lib as L
L.lib().sh_set_launch_mode(L.context(0), a.hostloop)
cols = generate(a.kind, a.n, 0)
d = tuple(torch.from_numpy(c).cuda() for c in cols)
f = P.hull_indices_2d if len(d) == 2 else P.hull_indices_3d
for _ in range(a.reps):
    idx = f(d)
    torch.cuda.synchronize()
print("h", idx.numel(), "trace", P.trace().tolist()[:30])

"""racecheck run: host-driven round loop (launch mode 1, no conditional
graph) and no facets (the persistent facet kernel spin-waits on other warps,
which racecheck's serialised execution can not make progress on)."""
import os, sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from paper_1201_2936_b200.datagen import generate
_lib.lib().sh_set_launch_mode(_lib.context(0), 1)
for kind, n in [("uniform-disk", 20000), ("on-circle", 3000)]:
    P.hull_indices_2d(tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 1)))
for kind, n in [("uniform-ball", 5000), ("unit-cube", 3000)]:
    P.hull_indices_3d(tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 1)))
torch.cuda.synchronize()
print("done")

"""Small end-to-end run for compute-sanitizer (memcheck): 2D/3D hulls,
facets, forced long rounds, device generation."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import pointio
from paper_1201_2936_b200.datagen import generate
for kind, n in [("uniform-disk", 20000), ("on-circle", 3000), ("unit-square", 5000)]:
    cols = tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 1))
    P.hull_indices_2d(cols)
for kind, n in [("uniform-ball", 20000), ("on-sphere", 2000), ("unit-cube", 5000)]:
    cols = tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 1))
    P.hull_indices_3d(cols, facets=True)
os.environ["SH_LONG_MIN_LIVE"] = "0"; os.environ["SH_LONG_SEG_MIN"] = "1"
P.hull_indices_2d(tuple(torch.from_numpy(c).cuda() for c in generate("on-circle", 900, 2)))
P.hull_indices_3d(tuple(torch.from_numpy(c).cuda() for c in generate("uniform-ball", 20000, 2)))
pointio.generate_device("unit-cube", 1000, 3)
torch.cuda.synchronize()
print("done")

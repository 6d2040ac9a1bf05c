import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
for kind, n in (("uniform-ball", 10_000_000), ("unit-cube", 10_000_000), ("uniform-ball", 200_000_000)):
    d = tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 0))
    P.hull_indices_3d(d); torch.cuda.synchronize()
    print(kind, n, P.filter_stats())
    del d; torch.cuda.empty_cache()

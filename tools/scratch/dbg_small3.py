import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
cols = generate(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
f = P.hull_indices_2d if len(cols) == 2 else P.hull_indices_3d
print(f(tuple(torch.from_numpy(c).cuda() for c in cols)).numel())

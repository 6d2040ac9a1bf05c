"""Run one C2 hull in launch mode 1 (host loop) so ncu sees each kernel."""
import sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from paper_1201_2936_b200.datagen import generate
kind = sys.argv[1] if len(sys.argv) > 1 else "uniform-disk"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
cols = generate(kind, n, 0)
d = tuple(torch.from_numpy(c).cuda() for c in cols)
f = P.hull_indices_2d if len(cols) == 2 else P.hull_indices_3d
f(d)
_lib.lib().sh_set_launch_mode(_lib.context(0), 1)
f(d)
torch.cuda.synchronize()

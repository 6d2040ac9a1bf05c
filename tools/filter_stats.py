"""3D filter diagnostics on the C4 ball / cube and C5 clouds (sh_filter_stats;
run with SH_LIB pointing at a -DSH_FILTER_CYCLES build for the cycle and
per-item histograms)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
for kind, n in (("uniform-ball", 10_000_000), ("unit-cube", 10_000_000), ("uniform-ball", 200_000_000)):
    d = tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 0))
    P.hull_indices_3d(d); torch.cuda.synchronize()
    fs = P.filter_stats()
    hist = {k: v for k, v in fs.items() if k.startswith("item_cyc_2^") and v}
    print(kind, n, {k: v for k, v in fs.items() if not k.startswith("item_cyc_2^")})
    print("   k_f_test items by wall cycles:", hist)
    del d; torch.cuda.empty_cache()

import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, torch, oracle, paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
bad = 0
for kind,n,seed in [('uniform-disk',2_000_000,1),('on-circle',300_000,2),('near-circle',500_000,3),('unit-square',1_000_000,4),
                    ('uniform-ball',500_000,1),('unit-cube',300_000,2),('on-sphere',20_000,3),('near-sphere',100_000,4)]:
    cols=generate(kind,n,seed)
    d=tuple(torch.from_numpy(c).cuda() for c in cols)
    if len(cols)==2:
        idx,res=P.hull_indices_2d(d, return_info=True); o=oracle.hull2d(*cols); oi=o.idx
        ok = np.array_equal(idx.cpu().numpy(), oi) and res.iterations==o.iterations and np.array_equal(P.trace()[:, :3], o.trace)
    else:
        idx,_,res=P.hull_indices_3d(d, return_info=True); o,oi,_=oracle.full_hull3d(*cols)
        ok = np.array_equal(np.sort(idx.cpu().numpy()),np.sort(oi)) and res.iterations==o.iterations and res.candidates==len(o.idx)
    bad += not ok
    print(kind, n, 'OK' if ok else 'MISMATCH', flush=True)
print("ALL OK" if not bad else f"{bad} MISMATCHES")

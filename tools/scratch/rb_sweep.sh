for cfg in "128 4" "128 8" "256 4"; do
  set -- $cfg
  make -s -C paper_1201_2936_b200/csrc clean; make -s -C paper_1201_2936_b200/csrc EXTRA="-DF_LOCAL_N=6 -DSH_RB=$1 -DSH_RITEMS=$2" || { echo "build fail $cfg"; continue; }
  echo "RB=$1 RITEMS=$2"; timeout 200 python tools/round_probe.py uniform-disk 2>&1 | head -6
  timeout 100 python -c "
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, torch, oracle, paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
for kind,n in [('uniform-disk',2_000_000),('on-circle',300_000),('uniform-ball',500_000)]:
    cols=generate(kind,n,1)
    d=tuple(torch.from_numpy(c).cuda() for c in cols)
    if len(cols)==2:
        idx=P.hull_indices_2d(d).cpu().numpy(); o=oracle.hull2d(*cols)
    else:
        idx=P.hull_indices_3d(d).cpu().numpy(); o,o2,_=oracle.full_hull3d(*cols); o.idx=o2
    print(kind, 'OK' if np.array_equal(np.sort(idx),np.sort(o.idx)) else 'MISMATCH')
"
done

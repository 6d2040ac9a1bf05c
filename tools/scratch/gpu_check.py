"""Ad-hoc GPU bring-up check: GPU hull vs the C oracle on many inputs."""
import sys, time, traceback
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import oracle
import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate

def run2(kind, n, seed):
    x, y = generate(kind, n, seed)
    o = oracle.hull2d(x, y)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    torch.cuda.synchronize()
    t = time.time()
    idx, res = P.hull_indices_2d((dx, dy), return_info=True)
    torch.cuda.synchronize()
    dt = time.time() - t
    g = np.sort(idx.cpu().numpy())
    ok = np.array_equal(g, np.sort(o.idx)) and res.iterations == o.iterations
    tr = P.trace()
    trok = np.array_equal(tr[:, :3], o.trace) if ok else None
    return ok, trok, len(g), len(o.idx), res.iterations, o.iterations, dt

def run3(kind, n, seed):
    x, y, z = generate(kind, n, seed)
    o = oracle.hull3d(x, y, z)
    d = tuple(torch.from_numpy(c).cuda() for c in (x, y, z))
    try:
        idx, fac, res = P.hull_indices_3d(d, return_info=True)
    except Exception as e:
        return ("exc", repr(e), o.status)
    g = np.sort(idx.cpu().numpy())
    ok = np.array_equal(g, np.sort(o.idx)) and res.iterations == o.iterations
    tr = P.trace()
    trok = np.array_equal(tr[:, :3], o.trace) and np.array_equal(tr[:, 3], o.flat_counts[:len(tr)])
    return ok, trok, len(g), len(o.idx), res.iterations, o.iterations

bad = 0
for kind in ["unit-square", "uniform-disk", "on-circle", "near-circle"]:
    for n in [1, 2, 3, 4, 5, 16, 100, 1000, 5000, 100000]:
        for seed in range(3):
            try:
                r = run2(kind, n, seed)
            except Exception:
                traceback.print_exc(); r = (False,)
            if not r[0] or not r[1]:
                bad += 1; print("2D FAIL", kind, n, seed, r, flush=True)
print("2D small done, bad =", bad, flush=True)
for kind, n in [("unit-square", 10**6), ("uniform-disk", 10**7), ("on-circle", 10**6), ("near-circle", 10**6)]:
    r = run2(kind, n, 0)
    print("2D big", kind, n, r, flush=True)
bad3 = 0
for kind in ["unit-cube", "uniform-ball", "on-sphere", "near-sphere"]:
    for n in [1, 2, 3, 4, 8, 32, 100, 1000, 20000]:
        for seed in range(3):
            try:
                r = run3(kind, n, seed)
            except Exception:
                traceback.print_exc(); r = (False,)
            if r[0] is not True or r[1] is not True:
                bad3 += 1; print("3D FAIL", kind, n, seed, r, flush=True)
print("3D small done, bad =", bad3, flush=True)
for kind, n in [("unit-cube", 10**6), ("uniform-ball", 10**6)]:
    print("3D big", kind, n, run3(kind, n, 0), flush=True)
# timing: disk 100M resident
x, y = generate("uniform-disk", 10**8, 0)
dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for it in range(4):
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); idx = P.hull_indices_2d((dx, dy)); e.record(); torch.cuda.synchronize()
    print("disk100M ms", s.elapsed_time(e), "h", idx.numel(), flush=True)

"""Where does a small synchronous hull call spend its time?"""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import _lib
from paper_1201_2936_b200.datagen import generate
n = int(sys.argv[1])
d = tuple(torch.from_numpy(c).cuda() for c in generate("uniform-disk", n, 0))
L, ctx = _lib.lib(), _lib.context(0)
P.hull_indices_2d(d); torch.cuda.synchronize()
out = torch.empty(n + 2, dtype=torch.int64, device="cuda")
res = _lib.ShResult(); sp = torch.cuda.current_stream().cuda_stream
def t(f, k=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return round((time.perf_counter() - t0) / k * 1e3, 3)
nan = float("nan")
print("n", n)
print("public api", t(lambda: P.hull_indices_2d(d)))
print("sync abi", t(lambda: L.sh_hull2d(ctx, d[0].data_ptr(), d[1].data_ptr(), 1, n, 1e-12, nan, out.data_ptr(), ctypes.byref(res), sp)))
print("async abi", t(lambda: L.sh_hull2d_async(ctx, d[0].data_ptr(), d[1].data_ptr(), 1, n, 1e-12, nan, out.data_ptr(), sp)))
print("async+fetch", t(lambda: (L.sh_hull2d_async(ctx, d[0].data_ptr(), d[1].data_ptr(), 1, n, 1e-12, nan, out.data_ptr(), sp), L.sh_fetch(ctx, ctypes.byref(res), sp))))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [L.sh_hull2d_async(ctx, d[0].data_ptr(), d[1].data_ptr(), 1, n, 1e-12, nan, out.data_ptr(), sp) for _ in range(20)]; e1.record(); torch.cuda.synchronize()
print("device per hull", round(e0.elapsed_time(e1) / 20, 3))

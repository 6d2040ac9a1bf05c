"""Time the stages of one sharded hull step (world of 1, NCCL) on C2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_1201_2936_b200 import sharded
from paper_1201_2936_b200.datagen import generate
import paper_1201_2936_b200 as P
kind = sys.argv[1] if len(sys.argv) > 1 else "uniform-disk"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000
d = tuple(torch.from_numpy(c).cuda() for c in generate(kind, n, 0))
for _ in range(3): sharded.hull_sharded(d, 0)
torch.cuda.synchronize()
T = {}
def tick(name, t0):
    torch.cuda.synchronize(); T[name] = T.get(name, 0) + (time.perf_counter() - t0) * 1e3; return time.perf_counter()
for _ in range(5):
    t = time.perf_counter()
    st = sharded.device_stats(d, 0); t = tick("stats", t)
    g = sharded.device_reduce_stats(sharded._all_gather(st, None), len(d)); t = tick("gather+reduce", t)
    gidx, coords, eps = sharded.device_hull(d, 0, P.Tolerance(), g); t = tick("local hull", t)
    rec = torch.cat([coords, gidx.to(torch.float64)[:, None]], dim=1)
    cs = torch.tensor([rec.shape[0], 0], dtype=torch.int64, device="cuda"); al = sharded._all_gather(cs, None).cpu().tolist(); t = tick("counts", t)
    parts = sharded._all_gather(rec, None); t = tick("records", t)
    u = parts[0]; dim = len(d)
    u = u[torch.argsort(u[:, dim])]; keep = torch.ones(u.shape[0], dtype=torch.bool, device=u.device); keep[1:] = u[1:, dim] != u[:-1, dim]; u = u[keep]; t = tick("merge prep", t)
    cols = tuple(u[:, k].contiguous() for k in range(dim)); t = tick("merge cols", t)
    idx = sharded.device_merge_hull(cols, P.Tolerance(eps_abs=eps)); t = tick("merge hull", t)
    f = P.hull_indices_2d if dim == 2 else P.hull_indices_3d
    f(cols); t = tick("small hull again", t)
    f = P.hull_indices_2d if len(d) == 2 else P.hull_indices_3d
    f(d); t = tick("plain hull", t)
print({k: round(v / 5, 3) for k, v in T.items()})
dist.destroy_process_group()

import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_1201_2936_b200 as P
from paper_1201_2936_b200.datagen import generate
n = int(sys.argv[1]); mode = sys.argv[2]
if mode != "none":
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29556")
    if mode == "nccl_dev":
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("nccl", rank=0, world_size=1)
    x = torch.ones(4, device="cuda"); dist.all_reduce(x)
d = tuple(torch.from_numpy(c).cuda() for c in generate("uniform-disk", n, 0))
P.hull_indices_2d(d); torch.cuda.synchronize()
def t(f, k=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize(); return round((time.perf_counter() - t0) / k * 1e3, 3)
print(mode, n, "public api", t(lambda: P.hull_indices_2d(d)), "empty sync", t(lambda: torch.cuda.synchronize()))

"""Phase timing of the sharded pipeline at world size 1 (NCCL)."""
import os, sys, time
import torch, torch.distributed as dist
sys.path.insert(0, "/root/repo")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import paper_1201_2936_b200 as P
from paper_1201_2936_b200 import sharded
from paper_1201_2936_b200.datagen import generate
cols = tuple(torch.from_numpy(c).cuda() for c in generate("uniform-disk", 100_000_000, 0))
for _ in range(3):
    sharded.hull_sharded(cols, 0)
torch.cuda.synchronize()
import cProfile, pstats
t = time.perf_counter()
for _ in range(10):
    r = sharded.hull_sharded(cols, 0)
torch.cuda.synchronize()
print("sharded ms/step (wall):", (time.perf_counter() - t) * 100)
t = time.perf_counter()
for _ in range(10):
    r2 = P.hull_indices_2d(cols)
torch.cuda.synchronize()
print("plain ms/step (wall):", (time.perf_counter() - t) * 100)
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    sharded.hull_sharded(cols, 0)
torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
dist.destroy_process_group()

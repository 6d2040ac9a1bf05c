"""H2D throughput of 1.6 GB pinned -> device: one stream vs chunks over 2-4 streams."""
import time, torch
n = 100_000_000
host = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
dev = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(4)]
def run(ns, chunks):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for s in streams[:ns]:
        s.wait_stream(cur)
    k = 0
    for c in range(2):
        step = n // chunks
        for j in range(chunks):
            s = streams[k % ns]; k += 1
            with torch.cuda.stream(s):
                dev[c][j * step:(j + 1) * step].copy_(host[c][j * step:(j + 1) * step], non_blocking=True)
    for s in streams[:ns]:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for ns, ch in ((1, 1), (2, 1), (2, 2), (2, 8), (4, 4), (4, 16)):
    t = min(run(ns, ch) for _ in range(5))
    print(f"streams={ns} chunks/col={ch}: {t:.2f} ms  {1.6e9 / (t / 1e3) / 1e9:.1f} GB/s")

"""Benchmark of the B200 Quickhull hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]
                    [--scaling weak|strong]

A "step" is one whole hull of the configured workload: every Quickhull
round of it, from the first bbox/extreme pass to the last vertex, as ONE
CUDA-graph launch through the C ABI (the round loop runs on the device).

Default workload (N=1): BASELINE.json configs[1] = C2, 2D Quickhull of 100M
points uniform in the unit disk (fp64, reference generator, seed 0).  The
other configs are parity cases (tests/), selectable here with --config.

N GPUs (--gpus N): one process per GPU over NCCL.  Without a launcher
(WORLD_SIZE unset) bench.py starts its own N ranks through
torch.distributed.run.  Every rank hulls a contiguous slice with the whole
input's statistics exchanged by one NCCL all-gather, then the candidate
records are all-gathered and rank 0 hulls their union
(paper_1201_2936_b200/sharded.py).  --scaling weak (default; C5: strong):
each rank owns the configured n points (N*n in total); strong: the
configured n points in total, n/N per rank -- BASELINE config C5 is 200M
points total over 1/2/4/8 GPUs.  value = total points / max-rank time.

value     Mpoints/s = n * K / (device time of K hulls), input resident in HBM
          (1.6 GB, far larger than the 126 MB L2, so no flush is needed).
e2e       same metric through the public API with HOST (pinned) buffers:
          H2D copy of the points + hull + D2H of the vertex indices per step.
roofline  the round kernels: algorithmic bytes of each launch over its
          CUDA-event duration, measured in an event-instrumented pass
          (launch mode 2) right after the timed region; peak =
          MEASURED_PEAKS.json hbm_gbs.  Bytes per launch (R_d = 8*dim + 4):
          first split 8*dim*n (read only); round 1 8*dim*n + R_d*n_2 (it
          re-reads the input instead of a materialised split); round r >= 2
          R_d*(n_r + n_{r+1}).  whole_hull_frac uses SURVEY.md §8(d)'s
          canonical B_alg (materialised first split), which this design undercuts.
clocks    nvidia-ml samples every 2 ms through the warm-up, the timed region
          and a clock window of further steps (at least 1 s of load).
cpu_baseline  the oracle (single-threaded C restatement of the reference
          drivers; 3D: its loop + Qhull on the candidates standing in for the
          reference's LP filter) on the same workload, rank 0, N=1 only.

--impl reference: the reference's CPU implementation of the path -- here the
oracle port, since the reference is pure Python and cannot travel to the GPU
box -- on the same workload (the whole cloud when one run takes at most a few
seconds; otherwise a bounded prefix of it, marked same_config false), rank 0.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpoints/sec for 2D/3D hull (device-timed) at 1/2/4/8 B200; % HBM roofline"
UNIT = "Mpoints/s"

CONFIGS = {
    "C1": ("C1: 2D Quickhull, 1M points uniform in unit square (fp64)", "unit-square", 1_000_000),
    "C2": ("C2: 2D Quickhull, 100M points uniform in unit disk (fp64)", "uniform-disk", 100_000_000),
    "C3": ("C3: 2D Quickhull, 10M points on unit circle (fp64)", "on-circle", 10_000_000),
    "C3n": ("C3': 2D Quickhull, 10M points near unit circle, band 0.01 (fp64)", "near-circle",
            10_000_000),
    "C4c": ("C4: 3D Quickhull, 10M points uniform in unit cube (fp64)", "unit-cube", 10_000_000),
    "C4b": ("C4: 3D Quickhull, 10M points uniform in unit ball (fp64)", "uniform-ball", 10_000_000),
    "C5": ("C5: 3D Quickhull, 200M points uniform in ball (fp64)", "uniform-ball", 200_000_000),
}
# the reference arm hulls the whole cloud when the port needs at most a few
# seconds for it (C1-C4); C5 (200M 3D points, ~25 s per run) is sampled
REF_SAMPLE = {"C5": 20_000_000}

KID_ROUND_FIRST, KID_ROUND = 3, 4


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """SM clocks and throttle reasons sampled every 2 ms from a thread
    (nvidia-ml; nvidia-smi's 100 ms period is longer than a timed region)
    between start() and stop() (B200_PROFILING.md's clock record)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.run = False
        self.t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.t = None
            return
        self.run = True

        def loop():
            bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                    "sw_power_cap": 0x4}
            while self.run:
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                    self.rows.append((sm, [k for k, v in bits.items() if r & v], util))
                except Exception:
                    pass
                time.sleep(0.002)
        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()

    def stop(self):
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-ml unavailable"], "samples": 0}
        self.run = False
        self.t.join(timeout=2)
        sm = [r[0] for r in self.rows]
        reasons = sorted({x for r in self.rows for x in r[1]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.mx,
                "reasons": reasons, "samples": len(self.rows), "period_ms": 2}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(cfg):
    """ncu dram bytes per k_round launch from the committed full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "round_traffic.json")) as f:
            return json.load(f).get(cfg)
    except (OSError, ValueError):
        return None


def gen(kind, n, start=0):
    from paper_1201_2936_b200.datagen import generate
    return generate(kind, n, 0, start=start)


def measure_roofline(L, ctx, device, launch, n, dim, config, hull_ms):
    """roofline object of the round kernels: per-launch CUDA events (launch
    mode 2) around one hull run by ``launch()`` on ``ctx``; bytes per launch
    from the per-round trace."""
    import paper_1201_2936_b200 as P
    L.sh_set_launch_mode(ctx, 2)
    per = []
    for _ in range(3):
        launch()
        import torch
        torch.cuda.synchronize()
        kinds = np.zeros(4096, np.int32)
        ms = np.zeros(4096, np.float32)
        k = L.sh_launch_times(ctx, kinds.ctypes.data, ms.ctypes.data, 4096)
        per.append((kinds[:k].copy(), ms[:k].copy()))
    L.sh_set_launch_mode(ctx, 0)
    tr = P.trace(device)  # of the hull just measured
    Rd = 8 * dim + 4
    n1 = int(tr[0, 0]) if len(tr) else 0
    # bytes each round launch must move in this design: the first split
    # reads the input and writes nothing; round 1 re-reads the input (the
    # split is re-derived on the fly) and writes its survivors; later rounds
    # read and write R_d-byte records
    round_bytes = [8 * dim * n]
    for r, (a, b, _, _) in enumerate(tr):
        round_bytes.append((8 * dim * n if r == 0 else Rd * int(a)) + Rd * int(b))
    # SURVEY.md §8(d)'s canonical B_alg (materialised first split)
    b_alg = 2 * 8 * dim * n + Rd * n1 + sum(Rd * (int(a) + int(b)) for a, b, _, _ in tr)
    best = None
    kernel_ms_by_kind = {}
    for kinds, ms in per:
        rt = ms[(kinds == KID_ROUND_FIRST) | (kinds == KID_ROUND)]
        if len(rt) != len(round_bytes):
            continue
        tot_round = float(rt.sum())
        if best is None or tot_round < best[0]:
            best = (tot_round, float(ms.sum()), rt)
            names = ["init", "first_reduce", "line_far", "round_first", "round", "book", "filter",
                     "output", "facets"]
            kernel_ms_by_kind = {names[k]: round(float(ms[kinds == k].sum()), 4)
                                 for k in sorted(set(kinds.tolist()))}
    if not best:
        return None
    peak, peak_src = measured_peak()
    tot_round, tot_all, rt = best
    launches = len(round_bytes)
    achieved = sum(round_bytes) / launches / (tot_round / launches / 1e3) / 1e9
    return {"bound": "hbm",
            "kernel": "k_round1 (round 1, fused with the first split) + k_round (rounds >= 2): "
                      "discard+classify+regroup+argmax",
            "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": committed_traffic(config),
            "peak_source": peak_src, "launches": launches,
            "algorithmic_bytes_per_launch": int(sum(round_bytes) / launches),
            "avg_launch_ms": round(tot_round / launches, 4),
            "share_of_kernel_time": round(tot_round / tot_all, 3),
            "whole_hull_frac": round(b_alg / (hull_ms / 1e3) / 1e9 / peak, 4),
            "whole_hull_b_alg_bytes": b_alg,
            "design_bytes_per_hull": sum(round_bytes) + 8 * dim * n,
            "per_round_gbs": [round(float(b / (t / 1e3) / 1e9), 1) for b, t in zip(round_bytes, rt)],
            "kernel_ms_by_kind": kernel_ms_by_kind}


def clock_window(clk, step, seconds=1.0):
    """Keep the GPU busy with more (untimed) steps so the clock record covers
    at least ``seconds`` of load."""
    import torch
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        step()
        torch.cuda.synchronize()
    return clk.stop()


def run_sharded(args, ws, rank, local):
    """N GPUs: rank r hulls a contiguous slice of the cloud; the global hull
    is assembled by paper_1201_2936_b200.sharded (one NCCL all-gather of the
    slices' statistics -> global eps and first split on the device, the
    local hulls, an all-gather of the candidate records, the rank-0 merge).
    weak: n points per rank (N*n total); strong: n points in total.
    value = total points / max-rank time."""
    import torch
    import torch.distributed as dist
    from paper_1201_2936_b200 import sharded

    desc, kind, n = CONFIGS[args.config]
    scaling = args.scaling or ("strong" if args.config == "C5" else "weak")
    n_total = n if scaling == "strong" else n * ws
    b0, b1 = (n_total * rank) // ws, (n_total * (rank + 1)) // ws
    cols = gen(kind, b1 - b0, start=b0)
    dim = len(cols)
    host = tuple(torch.from_numpy(c).pin_memory() for c in cols)
    d = tuple(h.to("cuda", non_blocking=True) for h in host)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    def step(inp):
        return sharded.hull_sharded(inp, b0, return_info=True)

    clk = Clocks(local)
    clk.start()
    for _ in range(args.warmup):
        res, info = step(d)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    dist.barrier()
    torch.cuda.synchronize()
    ev[0].record(stream)
    for i in range(args.steps):
        res, info = step(d)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clocks = clock_window(clk, lambda: step(d))
    tot = torch.tensor([sum(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))],
                       dtype=torch.float64, device="cuda")
    dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    tot_ms = float(tot.item())
    value = n_total * args.steps / (tot_ms / 1e3) / 1e6
    # e2e: pinned host slices in (copied into one set of device buffers,
    # allocated once), global indices out on rank 0
    e2e_ms = []
    dd = tuple(torch.empty_like(x) for x in d)
    for i in range(min(args.steps, 5) + 2):
        dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for a, h in zip(dd, host):
            a.copy_(h, non_blocking=True)
        r, _ = step(dd)
        hout = r.cpu() if r is not None else None
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i >= 2:  # two warm-up copies (first-touch of the pinned pages)
            e2e_ms.append(float(t.item()))
    e2e_val = n_total / (statistics.mean(e2e_ms) / 1e3) / 1e6
    # round-kernel roofline of this rank's local hull (same kernels as N=1,
    # with the global eps), measured on rank 0
    roofline = None
    if rank == 0:
        from paper_1201_2936_b200 import _lib
        import paper_1201_2936_b200 as P
        L, ctx = _lib.lib(), _lib.context(local)
        f = P.hull_indices_2d if dim == 2 else P.hull_indices_3d
        tol = P.Tolerance(eps_abs=info["eps"])
        roofline = measure_roofline(L, ctx, local, lambda: f(d, tol), b1 - b0, dim, args.config,
                                    tot_ms / args.steps)
    launches = None
    if roofline:
        # per rank and step: the local hull's graph (as in main(); with more
        # than one rank also stage 1 / 2 and the statistics reduction), rank
        # 0's merge hull of the gathered candidates not counted
        r = roofline["launches"] - 1
        long_peel = 5
        launches = args.steps * ((2 if ws > 1 else 0) + 4 + (1 if dim == 3 else 0) + 2 + 3 * long_peel
                                 + 2 * max(0, r - 1 - long_peel) + (14 if dim == 3 else 1))
    if rank == 0:
        h = int(res.numel())
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(tot_ms / args.steps, 4), "higher_is_better": True,
                "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc + (f", {n_total:,} points over {ws} GPU(s) (strong scaling)"
                                               if scaling == "strong" else
                                               f", x{ws} ranks: {n:,} points per GPU (weak scaling)"),
                           "n_total": n_total, "n_per_gpu": b1 - b0, "dim": dim, "hull": h,
                           "union_candidates": info["union"],
                           "l2": "inputs larger than the 126 MB L2; no flush",
                           "parallelism": f"dp{ws}: contiguous index slices; one NCCL all-gather of the "
                                          "slice statistics (bbox + lexicographic extremes) -> global eps "
                                          "and first split on the device; all-gather of the candidate "
                                          "records; rank-0 merge hull"},
                "e2e": {"value": round(e2e_val, 2), "unit": UNIT,
                        "h2d_bytes_per_step": 8 * dim * n_total, "d2h_bytes_per_step": 8 * h,
                        "ms_per_step": round(statistics.mean(e2e_ms), 3)},
                "gpu_launches": launches, "roofline": roofline, "cpu_baseline": None, "clocks": clocks}
        print(json.dumps(line), flush=True)


def reference_run(dim, cols):
    """One run of the CPU reference port on ``cols``: the oracle's 2D driver,
    or its 3D loop + Qhull on the candidates (the stand-in for the
    reference's LP filter)."""
    import oracle
    if dim == 2:
        r = oracle.hull2d(*cols)
    else:
        r = oracle.full_hull3d(*cols)[0]
    assert r.status == 0
    return r


def run_reference(args, rank):
    if rank != 0:
        return
    desc, kind, n = CONFIGS[args.config]
    m = min(n, REF_SAMPLE.get(args.config, n))
    cols = gen(kind, m)
    dim = len(cols)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        reference_run(dim, cols)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = m * len(times) / tot / 1e6
    what = ("the whole cloud" if m == n else f"the first {m:,} points of the cloud (same generator/seed)")
    sample = (f"{what} per step; single-threaded C restatement of the reference drivers "
              f"(oracle/qh_oracle.c)" + ("" if dim == 2 else "; 3D: its loop + Qhull on the candidates "
                                         "standing in for the reference's LP filter"))
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * tot / len(times), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "n": m, "same_config": m == n, **({} if m == n else {"sample_of": n})},
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n):
    """bench.py --gpus N without a launcher: run N ranks of this script
    through torch.distributed.run (one process per GPU) and pass rank 0's
    line through."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ, SH_BENCH_CHILD="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--facets", action="store_true",
                    help="3D configs: also build the facet triples inside every step")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (sharded) pipeline even at N=1 (C5 always does)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="multi-GPU work split (default: strong for C5, weak otherwise)")
    args = ap.parse_args()
    ws, rank, local = dist_env()

    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.gpus > 1 and ws == 1 and not os.environ.get("SH_BENCH_CHILD"):
        sys.exit(spawn_ranks(args.gpus))

    import torch
    import torch.distributed as dist
    import ctypes

    import paper_1201_2936_b200 as P
    from paper_1201_2936_b200 import _lib

    torch.cuda.set_device(local)
    if ws > 1 or args.sharded or args.config == "C5":
        # NCCL's log (communicator ranks, NVLS/NVLink paths) goes to stderr:
        # rank 0 prints one JSON line on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_sharded(args, ws, rank, local)
        dist.destroy_process_group()
        return

    def barrier():
        if ws > 1:
            dist.barrier()

    desc, kind, n = CONFIGS[args.config]
    cols = gen(kind, n)
    dim = len(cols)
    host = tuple(torch.from_numpy(c).pin_memory() for c in cols)
    d = tuple(h.to("cuda", non_blocking=True) for h in host)
    torch.cuda.synchronize()
    L, ctx = _lib.lib(), _lib.context(local)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    want_fac = args.facets and dim == 3
    fcap = 4 * n + 8 if want_fac else 0  # n is at most 2^28 here; cap covers 2*candidates
    fac = torch.empty((max(min(fcap, 1 << 24), 1), 3), dtype=torch.int32, device="cuda")
    fcap = min(fcap, 1 << 24)
    res = _lib.ShResult()
    ptrs = [t.data_ptr() for t in d]
    nan = float("nan")

    def launch():
        if dim == 2:
            rc = L.sh_hull2d_async(ctx, ptrs[0], ptrs[1], 1, n, 1e-12, nan, out.data_ptr(), sp)
        else:
            rc = L.sh_hull3d_async(ctx, ptrs[0], ptrs[1], ptrs[2], 1, n, 1e-12, nan, out.data_ptr(),
                                   fac.data_ptr() if want_fac else None, fcap, sp)
        if rc:
            raise RuntimeError(_lib.last_error())

    # sync API once: sizes the segment tables (overflow retries happen here)
    if dim == 2:
        f = P.hull_indices_2d
    else:
        def f(pts):
            r = P.hull_indices_3d(pts, facets=want_fac)
            return r[0] if want_fac else r
    f(d)
    clk = Clocks(local)
    clk.start()
    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize()
    assert L.sh_fetch(ctx, ctypes.byref(res), sp) == 0
    rounds, h = int(res.iterations), int(res.h)

    # ---------------- timed region: K whole hulls, device-timed
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    torch.cuda.synchronize()
    ev[0].record(stream)
    for i in range(args.steps):
        launch()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clock_window(clk, launch)
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    tot_ms = sum(step_ms)
    if ws > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    assert L.sh_fetch(ctx, ctypes.byref(res), sp) == 0
    assert int(res.h) == h and int(res.iterations) == rounds
    value = n * ws * args.steps / (tot_ms / 1e3) / 1e6
    # the hull graph's kernel launches: init, first reduce, [3D: line-far],
    # first-split count, its book; round 1 (k_stream) and its book; LONG_PEEL
    # peeled round bodies outside the WHILE node, each (k_stream, k_round,
    # k_book) whether or not rounds are left (csrc/sh_common.cuh
    # SH_LONG_PEEL); (k_round, k_book) per WHILE iteration; then k_output
    # (2D) or the 14 filter kernels (3D); facets: 9 kernels
    long_peel = 5
    launches_per_hull = (4 + (1 if dim == 3 else 0) + 2 + 3 * long_peel + 2 * max(0, rounds - 1 - long_peel)
                         + (14 if dim == 3 else 1) + (9 if want_fac else 0))

    # ---------------- per-kernel pass (events after every launch)
    roofline = measure_roofline(L, ctx, local, launch, n, dim, args.config, tot_ms / args.steps)

    # ---------------- e2e: public API, pinned host buffers in, indices out
    e2e_ms = []
    for i in range(min(args.steps, 5) + 1):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        idx_host = f(host)
        e1.record(stream)
        torch.cuda.synchronize()
        if i:
            e2e_ms.append(e0.elapsed_time(e1))
    e2e_val = n * ws / (statistics.mean(e2e_ms) / 1e3) / 1e6
    assert idx_host.numel() == h

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        t0 = time.perf_counter()
        reference_run(dim, cols)
        dt = time.perf_counter() - t0
        cpu = {"value": round(n / dt / 1e6, 3), "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"the whole {args.config} workload ({n:,} points), one run, "
                         "single-threaded C restatement of the reference drivers (oracle/)" +
                         ("" if dim == 2 else "; 3D: its loop + Qhull on the candidates standing in "
                                              "for the reference's LP filter")}

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(tot_ms / args.steps, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc + (" + facet triples" if want_fac else ""), "n": n,
                           "dim": dim, "rounds": rounds, "hull": h,
                           "candidates": int(res.candidates), "eps_rel": 1e-12,
                           "facets": int(res.facets) if want_fac else None,
                           "l2": "inputs (%.1f GB) larger than the 126 MB L2; no flush" %
                                 (8 * dim * n / 1e9),
                           "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
                "e2e": {"value": round(e2e_val, 2), "unit": UNIT,
                        "h2d_bytes_per_step": 8 * dim * n, "d2h_bytes_per_step": 8 * h,
                        "ms_per_step": round(statistics.mean(e2e_ms), 3)},
                "gpu_launches": launches_per_hull * args.steps,
                "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
